"""B200-native (sm_100a) render path of Nexels (arXiv 2512.13796).

Drop-in for the reference's ``nexel::render`` / ``collection_pass`` /
``texturing_pass`` (proj/core/include/nexel/renderer.hpp). The compute runs in
``libnexel_b200.so`` (hand-written CUDA for sm_100a behind the C-ABI in
``include/nexel_b200.h``); this package is the host-side mirror of the
reference interface.
"""
from .api import (Camera, band_camera, image_bands, DeviceFrame, DeviceScene, FrameBuffers, HashGridConfig, NexelError, RenderResult,
                  LossWeights, Optimizer, RenderSettings, Renderer, Scene, SceneGrads, TextureField, UpstreamGrads, collection_pass, render,
                  losses_backward, render_backward, ring_camera, stump_like, texturing_pass)
from . import _abi

__all__ = [
    "Camera", "band_camera", "image_bands", "DeviceFrame", "DeviceScene", "FrameBuffers", "HashGridConfig", "NexelError", "RenderResult",
    "LossWeights", "Optimizer", "RenderSettings", "Renderer", "Scene", "SceneGrads", "TextureField", "UpstreamGrads", "collection_pass",
    "losses_backward", "render", "render_backward", "ring_camera", "stump_like", "texturing_pass", "_abi",
]
