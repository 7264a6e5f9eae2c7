"""Python mirror of the reference render interface (nexel::render & co).

Same names, argument meaning and error behaviour as the reference's
``proj/core/include/nexel/renderer.hpp`` (render / collection_pass /
texturing_pass), ``scene.hpp`` (RenderSettings, Scene), ``camera.hpp``
(Camera), ``framebuffers.hpp`` (FrameBuffers) and ``error.hpp`` (Error with a
machine-readable code). Every call runs on the sm_100a library through the
C-ABI (include/nexel_b200.h); nothing here computes pixels.

Two layers:
  * ``Renderer`` — device-resident API: upload a Scene once, render cameras into
    device frames, download explicitly (what the benchmark times);
  * ``render`` / ``collection_pass`` / ``texturing_pass`` — the reference's
    value-semantics API returning host FrameBuffers (fp64 like the reference).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import hashlib
import math
from typing import Optional, Sequence

import numpy as np

from . import _abi


class NexelError(RuntimeError):
    """nexel::Error (error.hpp:10-22): ``code`` is "bad-settings", "bad-camera",
    "bad-primitive", or a boundary code ("cuda-error", "unsupported", ...)."""

    def __init__(self, code: str, message: str):
        super().__init__(message)
        self.code = code

    def __str__(self):
        return f"{self.code}: {self.args[0]}"


@dataclasses.dataclass
class RenderSettings:
    """RenderSettings (scene.hpp:10-21)."""
    top_k: int = 2
    background: Sequence[float] = (0.0, 0.0, 0.0)
    near_eps: float = 1e-3
    alpha_max: float = 0.999
    min_transmittance: float = 1e-4
    tile: int = 16
    no_gamma: bool = False
    no_prim_sh: bool = False
    no_downweight: bool = False
    # not a reference knob: NX_PRECISION_F64 renders the colours at the reference's fp64
    # precision (fp64 SH / hash grid / decoder); the default keeps fp32 colour and the
    # bf16x3 tensor-core decoder (decisions, depths and weights are fp64 either way)
    precision: int = 0

    def to_c(self) -> _abi.nx_settings:
        s = _abi.nx_settings()
        s.top_k = int(self.top_k)
        s.tile = int(self.tile)
        for i in range(3):
            s.background[i] = float(self.background[i])
        s.near_eps = float(self.near_eps)
        s.alpha_max = float(self.alpha_max)
        s.min_transmittance = float(self.min_transmittance)
        s.no_gamma = int(bool(self.no_gamma))
        s.no_prim_sh = int(bool(self.no_prim_sh))
        s.no_downweight = int(bool(self.no_downweight))
        s.precision = int(self.precision)
        return s

    @classmethod
    def from_c(cls, s: _abi.nx_settings) -> "RenderSettings":
        return cls(top_k=s.top_k, background=tuple(s.background), near_eps=s.near_eps, alpha_max=s.alpha_max,
                   min_transmittance=s.min_transmittance, tile=s.tile, no_gamma=bool(s.no_gamma),
                   no_prim_sh=bool(s.no_prim_sh), no_downweight=bool(s.no_downweight), precision=int(s.precision))


@dataclasses.dataclass
class HashGridConfig:
    """HashGridConfig (hash_grid.hpp:39-56)."""
    levels: int = 16
    log2_table: int = 20
    features: int = 2
    base_scale: float = 1.0
    growth: float = 2.0

    @classmethod
    def for_extent(cls, extent: float, levels: int = 16, log2_table: int = 20, features: int = 2):
        """HashGridConfig::for_extent (hash_grid.cpp:15-24)."""
        growth = math.pow(32768.0, 1.0 / (levels - 1)) if levels > 1 else 1.0
        return cls(levels, log2_table, features, 1.0 / extent, growth)

    def table_size(self) -> int:
        return 1 << self.log2_table

    def param_count(self) -> int:
        return self.levels * self.table_size() * self.features


@dataclasses.dataclass
class TextureField:
    """TextureField (texture_field.hpp:16-25): hash grid table [level][row][feature]
    and the bias-free MLP w1 [hidden][in], w2 [hidden][hidden], w3 [48][hidden]."""
    grid: HashGridConfig
    table: np.ndarray
    w1: np.ndarray
    w2: np.ndarray
    w3: np.ndarray
    n_hidden: int = 64

    def desc(self) -> _abi.nx_field_desc:
        d = _abi.nx_field_desc()
        d.levels = self.grid.levels
        d.log2_table = self.grid.log2_table
        d.features = self.grid.features
        d.n_hidden = self.n_hidden
        d.base_scale = self.grid.base_scale
        d.growth = self.grid.growth
        return d


@dataclasses.dataclass
class Scene:
    """Scene (scene.hpp:25-32): ``nexels`` is (N, 60) float64 in Nexel field order
    (primitive.hpp:21-28): mu[3], quat[4] (w,x,y,z), log_scale[2], opacity_raw,
    gamma_raw[2], sh[48]."""
    nexels: np.ndarray
    field: TextureField
    settings: RenderSettings = dataclasses.field(default_factory=RenderSettings)
    extent: float = 1.0

    def sh_degree(self) -> int:
        return 0 if self.settings.no_prim_sh else 3

    def fingerprint(self) -> str:
        h = hashlib.blake2b(digest_size=16)
        for a in (self.nexels, self.field.table, self.field.w1, self.field.w2, self.field.w3):
            a = np.ascontiguousarray(a, dtype=np.float64)
            h.update(str(a.shape).encode())
            h.update(a.view(np.uint8).data)
        h.update(repr(dataclasses.astuple(self.field.grid)).encode())
        h.update(str(self.field.n_hidden).encode())
        return h.hexdigest()


@dataclasses.dataclass
class Camera:
    """Camera (camera.hpp:17-43): pinhole, OpenCV axes, X_cam = R X_world + t."""
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    R: np.ndarray
    t: np.ndarray
    name: str = ""

    def to_c(self) -> _abi.nx_camera:
        c = _abi.nx_camera()
        c.width, c.height = int(self.width), int(self.height)
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        R = np.asarray(self.R, dtype=np.float64).reshape(9)
        t = np.asarray(self.t, dtype=np.float64).reshape(3)
        for i in range(9):
            c.R[i] = float(R[i])
        for i in range(3):
            c.t[i] = float(t[i])
        return c

    @classmethod
    def from_c(cls, c: _abi.nx_camera, name: str = "") -> "Camera":
        return cls(c.width, c.height, c.fx, c.fy, c.cx, c.cy, np.array(c.R[:], dtype=np.float64).reshape(3, 3),
                   np.array(c.t[:], dtype=np.float64), name)

    def position(self) -> np.ndarray:
        return -(np.asarray(self.R).T @ np.asarray(self.t))


@dataclasses.dataclass
class FrameBuffers:
    """FrameBuffers (framebuffers.hpp:61-86); slot layout pixel-major, slot-minor."""
    width: int
    height: int
    top_k: int
    base: np.ndarray
    ids: np.ndarray
    depths: np.ndarray
    weights: np.ndarray
    texture: np.ndarray
    final_img: np.ndarray
    residual: np.ndarray

    def pixel(self, x: int, y: int) -> int:
        return y * self.width + x

    def slot(self, pix: int, j: int) -> int:
        return pix * self.top_k + j


@dataclasses.dataclass
class RenderResult:
    """RenderResult (renderer.hpp:11-16)."""
    fb: FrameBuffers
    blended_error: np.ndarray


@dataclasses.dataclass
class UpstreamGrads:
    """UpstreamGrads (renderer.hpp:40-44): fp64 arrays in the FrameBuffers layouts
    (d_final H*W*3, d_weights H*W*K, d_texture H*W*K*3); None = zero."""
    d_final: Optional[np.ndarray] = None
    d_weights: Optional[np.ndarray] = None
    d_texture: Optional[np.ndarray] = None


@dataclasses.dataclass
class SceneGrads:
    """SceneGrads (renderer.hpp:31-36): ``prims`` (N, 60) PrimitiveGrad in Nexel field
    order (primitive.hpp:53-62) + FieldGrads (texture_field.hpp:41-47)."""
    prims: np.ndarray
    table: np.ndarray
    w1: np.ndarray
    w2: np.ndarray
    w3: np.ndarray

    @classmethod
    def allocate(cls, scene: "Scene") -> "SceneGrads":
        """SceneGrads::allocate (renderer.cpp:245-248): zeros shaped like the scene."""
        f = scene.field
        return cls(np.zeros((scene.nexels.shape[0], _abi.NX_PARAMS_PER_NEXEL)), np.zeros(f.grid.param_count()),
                   np.zeros(np.size(f.w1)), np.zeros(np.size(f.w2)), np.zeros(np.size(f.w3)))


@dataclasses.dataclass
class LossWeights:
    """LossWeights (losses.hpp:12-18)."""
    dssim: float = 0.2
    alpha: float = 0.005
    texture: float = 0.5
    opacity: float = 0.01
    grid: float = 0.01

    def to_c(self) -> _abi.nx_loss_weights:
        return _abi.nx_loss_weights(self.dssim, self.alpha, self.texture, self.opacity, self.grid)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_abi.PD)


def _f64(a, n: int, what: str):
    """Contiguous fp64 view of an optional host array of n values."""
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if a.size != n:
        raise NexelError("invalid-argument", f"{what}: expected {n} values, got {a.size}")
    return a


class DeviceScene:
    def __init__(self, renderer: "Renderer", handle: C.c_void_p, n: int):
        self.renderer = renderer
        self.handle = handle
        self.n = n

    def set_settings(self, settings: RenderSettings):
        s = settings.to_c()
        self.renderer._check(self.renderer.lib.nx_scene_set_settings(self.renderer.ctx, self.handle, C.byref(s)))

    def close(self):
        if self.handle:
            self.renderer.lib.nx_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceFrame:
    def __init__(self, renderer: "Renderer", handle: C.c_void_p):
        self.renderer = renderer
        self.handle = handle

    def view(self) -> _abi.nx_frame_view:
        v = _abi.nx_frame_view()
        self.renderer.lib.nx_frame_view_get(self.handle, C.byref(v))
        return v

    def set_backward(self, enable: bool = True):
        """Keep the fp64 base the reverse pass needs (nx_frame_set_backward)."""
        r = self.renderer
        r._check(r.lib.nx_frame_set_backward(r.ctx, self.handle, int(enable)))

    def base_f64(self) -> np.ndarray:
        """The fp64 base (Eq. 6) kept for render_backward."""
        v = self.view()
        out = np.empty(v.width * v.height * 3, np.float64)
        hf = _abi.nx_host_frame()
        hf.base_f64 = out.ctypes.data
        r = self.renderer
        r._check(r.lib.nx_frame_download(r.ctx, self.handle, C.byref(hf), None))
        r._check(r.lib.nx_ctx_synchronize(r.ctx))
        return out

    def upload(self, fb: "FrameBuffers"):
        """Host FrameBuffers (e.g. from ``render``) -> this device frame, fp64 base kept."""
        npix = fb.width * fb.height
        arrs = {
            "base": np.ascontiguousarray(fb.base, np.float32).reshape(-1),
            "ids": np.ascontiguousarray(fb.ids, np.int32).reshape(-1),
            "depths": np.ascontiguousarray(fb.depths, np.float64).reshape(-1),
            "weights": np.ascontiguousarray(fb.weights, np.float64).reshape(-1),
            "texture": np.ascontiguousarray(fb.texture, np.float32).reshape(-1),
            "final_img": np.ascontiguousarray(fb.final_img, np.float32).reshape(-1),
            "residual": np.ascontiguousarray(fb.residual, np.float32).reshape(-1),
            "base_f64": np.ascontiguousarray(fb.base, np.float64).reshape(-1),
        }
        if arrs["base"].size != npix * 3 or arrs["ids"].size != npix * fb.top_k:
            raise NexelError("invalid-argument", "FrameBuffers arrays do not match their shape")
        hf = _abi.nx_host_frame()
        for k, a in arrs.items():
            setattr(hf, k, a.ctypes.data)
        r = self.renderer
        r._check(r.lib.nx_frame_upload(r.ctx, self.handle, fb.width, fb.height, fb.top_k, C.byref(hf), None))
        r._check(r.lib.nx_ctx_synchronize(r.ctx))

    def stats(self) -> dict:
        st = _abi.nx_frame_stats()
        self.renderer._check(self.renderer.lib.nx_frame_stats_get(self.renderer.ctx, self.handle, C.byref(st)))
        return st.as_dict()

    def download(self, fields: Optional[Sequence[str]] = None) -> FrameBuffers:
        """Synchronous download into fresh numpy arrays (device-native dtypes)."""
        v = self.view()
        W, H, K = v.width, v.height, v.top_k
        out = {
            "base": np.empty((H * W * 3,), np.float32),
            "ids": np.empty((H * W * K,), np.int32),
            "depths": np.empty((H * W * K,), np.float64),
            "weights": np.empty((H * W * K,), np.float64),
            "texture": np.empty((H * W * K * 3,), np.float32),
            "final_img": np.empty((H * W * 3,), np.float32),
            "residual": np.empty((H * W,), np.float32),
        }
        want = set(fields) if fields else set(out)
        hf = _abi.nx_host_frame()
        for k, arr in out.items():
            setattr(hf, k, arr.ctypes.data if k in want else None)
        f64 = {}
        if fields and ("texture_f64" in want or "final_f64" in want):  # NX_PRECISION_F64 renders
            f64 = {"texture_f64": np.zeros((H * W * K * 3,)), "final_f64": np.zeros((H * W * 3,))}
            hf.texture_f64, hf.final_f64 = f64["texture_f64"].ctypes.data, f64["final_f64"].ctypes.data
        r = self.renderer
        r._check(r.lib.nx_frame_download(r.ctx, self.handle, C.byref(hf), None))
        r._check(r.lib.nx_ctx_synchronize(r.ctx))
        fb = FrameBuffers(W, H, K, **out)
        for k, v in f64.items():
            setattr(fb, k, v)
        return fb

    def close(self):
        if self.handle:
            self.renderer.lib.nx_frame_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Renderer:
    """One CUDA context (device + stream) of the sm_100a render path."""

    def __init__(self, device: int = 0):
        self.lib = _abi.load()
        self.ctx = C.c_void_p()
        st = self.lib.nx_ctx_create(int(device), C.byref(self.ctx))
        if st != _abi.NX_OK:
            raise NexelError(_abi.STATUS_CODES.get(st, "error"), f"cannot create a context on cuda:{device}")
        self.device = device

    def _check(self, status: int):
        if status != _abi.NX_OK:
            code = C.c_int()
            msg = self.lib.nx_ctx_last_error(self.ctx, C.byref(code)).decode()
            raise NexelError(_abi.STATUS_CODES.get(status, "error"), msg)

    @property
    def stream(self) -> int:
        return int(self.lib.nx_ctx_stream(self.ctx) or 0)

    def upload(self, scene: Scene) -> DeviceScene:
        nex = np.ascontiguousarray(scene.nexels, dtype=np.float64).reshape(-1, _abi.NX_PARAMS_PER_NEXEL)
        f = scene.field
        tab = np.ascontiguousarray(f.table, dtype=np.float64)
        w1 = np.ascontiguousarray(f.w1, dtype=np.float64)
        w2 = np.ascontiguousarray(f.w2, dtype=np.float64)
        w3 = np.ascontiguousarray(f.w3, dtype=np.float64)
        if tab.size != f.grid.param_count():
            raise NexelError("invalid-argument", "hash table size does not match the grid config")
        nin = f.grid.levels * f.grid.features
        if w1.size != f.n_hidden * nin or w2.size != f.n_hidden ** 2 or w3.size != 48 * f.n_hidden:
            raise NexelError("invalid-argument", "MLP weight shapes do not match the field")
        s = scene.settings.to_c()
        d = f.desc()
        h = C.c_void_p()
        self._check(self.lib.nx_scene_create(self.ctx, C.byref(s), nex.shape[0], _dp(nex), C.byref(d), _dp(tab),
                                             _dp(w1), _dp(w2), _dp(w3), C.byref(h)))
        return DeviceScene(self, h, nex.shape[0])

    def load_checkpoint(self, path: str):
        """load_checkpoint (checkpoint.hpp:27-28) straight into a device scene: returns
        (DeviceScene, info dict with iteration / extent / settings / field, cameras)."""
        h = C.c_void_p()
        info = _abi.nx_nexl_info()
        self._check(self.lib.nx_scene_load_nexl(self.ctx, str(path).encode(), C.byref(h), C.byref(info)))
        ds = DeviceScene(self, h, int(info.n_nexels))
        n = C.c_int(0)
        self._check(self.lib.nx_nexl_cameras(str(path).encode(), None, None, 0, C.byref(n)))
        cams = (_abi.nx_camera * max(n.value, 1))()
        names = (C.c_char * 64 * max(n.value, 1))()
        self._check(self.lib.nx_nexl_cameras(str(path).encode(), cams, names, n.value, C.byref(n)))
        cameras = [Camera.from_c(cams[i], bytes(names[i]).split(b"\0")[0].decode()) for i in range(n.value)]
        meta = {"iteration": int(info.iteration), "extent": float(info.extent), "n_nexels": int(info.n_nexels),
                "has_optimizer": bool(info.has_optimizer), "settings": RenderSettings.from_c(info.settings),
                "field": HashGridConfig(info.field.levels, info.field.log2_table, info.field.features,
                                        info.field.base_scale, info.field.growth), "n_hidden": info.field.n_hidden}
        return ds, meta, cameras

    def frame(self, width: int = 0, height: int = 0, top_k: int = 0) -> DeviceFrame:
        h = C.c_void_p()
        self._check(self.lib.nx_frame_create(self.ctx, width, height, top_k, C.byref(h)))
        return DeviceFrame(self, h)

    def collection_pass(self, dscene: DeviceScene, cam: Camera, frame: DeviceFrame, stream: int = 0):
        c = cam.to_c()
        self._check(self.lib.nx_collection_pass(self.ctx, dscene.handle, C.byref(c), frame.handle, stream or None))

    def texturing_pass(self, dscene: DeviceScene, cam: Camera, frame: DeviceFrame, stream: int = 0):
        c = cam.to_c()
        self._check(self.lib.nx_texturing_pass(self.ctx, dscene.handle, C.byref(c), frame.handle, stream or None))

    def render(self, dscene: DeviceScene, cam: Camera, frame: DeviceFrame, stream: int = 0):
        c = cam.to_c()
        self._check(self.lib.nx_render(self.ctx, dscene.handle, C.byref(c), frame.handle, stream or None))

    def render_views(self, dscene: DeviceScene, cams: Sequence[Camera], frames: Sequence[DeviceFrame],
                     stream: int = 0):
        """nx_render_views: cams[i] into frames[i % len(frames)], pipelined (asynchronous)."""
        arr = (_abi.nx_camera * len(cams))(*[c.to_c() for c in cams])
        fr = (C.c_void_p * len(frames))(*[f.handle for f in frames])
        self._check(self.lib.nx_render_views(self.ctx, dscene.handle, arr, len(cams), fr, len(frames),
                                             stream or None))

    def render_backward(self, dscene: DeviceScene, cam: Camera, frame: DeviceFrame, up: UpstreamGrads,
                        grads: SceneGrads, err_pixel: Optional[np.ndarray] = None,
                        blended_error: Optional[np.ndarray] = None):
        """render_backward (renderer.hpp:50-53) on host arrays: ACCUMULATES into
        ``grads`` (and ``blended_error`` when ``err_pixel`` is given). ``frame`` must
        hold the forward of ``cam`` rendered with ``frame.set_backward()`` enabled."""
        v = frame.view()
        npix, K = cam.width * cam.height, v.top_k
        d_final = _f64(up.d_final, npix * 3, "d_final")
        d_weights = _f64(up.d_weights, npix * K, "d_weights") if K else None
        d_texture = _f64(up.d_texture, npix * K * 3, "d_texture") if K else None
        u = _abi.nx_upstream()
        u.d_final = d_final.ctypes.data if d_final is not None else None
        u.d_weights = d_weights.ctypes.data if d_weights is not None else None
        u.d_texture = d_texture.ctypes.data if d_texture is not None else None
        arrs = [grads.prims, grads.table, grads.w1, grads.w2, grads.w3]
        for a in arrs:
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                raise NexelError("invalid-argument", "SceneGrads arrays must be C-contiguous float64")
        g = _abi.nx_grads()
        g.prims, g.table, g.w1, g.w2, g.w3 = (a.ctypes.data for a in arrs)
        err = _f64(err_pixel, npix, "err_pixel")
        if blended_error is not None and (blended_error.dtype != np.float64 or not blended_error.flags.c_contiguous):
            raise NexelError("invalid-argument", "blended_error must be C-contiguous float64")
        c = cam.to_c()
        self._check(self.lib.nx_render_backward_host(
            self.ctx, dscene.handle, C.byref(c), frame.handle, C.byref(u), C.byref(g),
            _dp(err) if err is not None else None,
            _dp(blended_error) if (blended_error is not None and err is not None) else None))

    def losses_backward(self, dscene: DeviceScene, frame: DeviceFrame, gt: np.ndarray, w: LossWeights,
                        grads: SceneGrads):
        """losses_backward (losses.hpp:52-56) on the device frame: returns (LossTerms
        dict, d_final, d_weights, d_texture); accumulates the opacity / grid terms into
        ``grads``."""
        v = frame.view()
        npix, K = v.width * v.height, v.top_k
        gt = _f64(gt, npix * 3, "gt")
        d_final, d_weights, d_texture = np.zeros(npix * 3), np.zeros(npix * K), np.zeros(npix * K * 3)
        for a in (grads.prims, grads.table):
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                raise NexelError("invalid-argument", "SceneGrads arrays must be C-contiguous float64")
        g = _abi.nx_grads(grads.prims.ctypes.data, grads.table.ctypes.data, None, None, None)
        t = _abi.nx_loss_terms()
        cw = w.to_c()
        self._check(self.lib.nx_losses_backward_host(self.ctx, dscene.handle, frame.handle, _dp(gt), C.byref(cw),
                                                     _dp(d_final), _dp(d_weights) if K else None,
                                                     _dp(d_texture) if K else None, C.byref(g), C.byref(t)))
        return t.as_dict(), d_final, d_weights, d_texture

    def download_scene(self, dscene: DeviceScene, field_like: TextureField):
        """The device scene's parameters in the reference's layouts: (nexels (N, 60),
        table, w1, w2, w3) as float64."""
        nex = np.zeros((dscene.n, _abi.NX_PARAMS_PER_NEXEL))
        arrs = [np.zeros(np.size(a)) for a in (field_like.table, field_like.w1, field_like.w2, field_like.w3)]
        self._check(self.lib.nx_scene_download(self.ctx, dscene.handle, _dp(nex), *(_dp(a) for a in arrs)))
        return (nex, *arrs)

    def optimizer(self, dscene: DeviceScene) -> "Optimizer":
        """fp64 Adam state for the device scene (nx_optimizer_create)."""
        return Optimizer(self, dscene)

    def pixel_error(self, frame: DeviceFrame, gt_device_ptr: int, err_device_ptr: int, stream: int = 0):
        """err[p] = sum_c |final - gt| / 3 on the device (trainer.cpp:288-295); device pointers."""
        self._check(self.lib.nx_pixel_error(self.ctx, frame.handle, C.c_void_p(gt_device_ptr),
                                            C.c_void_p(err_device_ptr), C.c_void_p(stream) if stream else None))

    def synchronize(self):
        self._check(self.lib.nx_ctx_synchronize(self.ctx))

    def set_profiling(self, on: bool):
        self._check(self.lib.nx_ctx_set_profiling(self.ctx, int(on)))

    def stage_times(self):
        """Mean per-stage device ms per frame since the last call (and the frame count)."""
        ms = (C.c_float * _abi.NX_NUM_STAGES)()
        frames = C.c_int(0)
        self._check(self.lib.nx_ctx_stage_times(self.ctx, ms, _abi.NX_NUM_STAGES, C.byref(frames)))
        return {name: float(ms[i]) for i, name in enumerate(_abi.STAGE_NAMES)}, frames.value

    # ---- parity / debug
    def tile_lists(self, dscene: DeviceScene, cam: Camera, reference_lists: bool = True):
        c = cam.to_c()
        total, tx, ty = C.c_int64(), C.c_int32(), C.c_int32()
        self._check(self.lib.nx_debug_tile_lists(self.ctx, dscene.handle, C.byref(c), int(reference_lists), None,
                                                 None, 0, C.byref(total), C.byref(tx), C.byref(ty)))
        n_tiles = tx.value * ty.value
        offsets = np.empty(n_tiles + 1, np.int64)
        ids = np.empty(max(total.value, 1), np.int32)
        self._check(self.lib.nx_debug_tile_lists(self.ctx, dscene.handle, C.byref(c), int(reference_lists),
                                                 offsets.ctypes.data_as(_abi.PI64), ids.ctypes.data_as(_abi.PI32),
                                                 total.value, C.byref(total), C.byref(tx), C.byref(ty)))
        return offsets, ids[: total.value], tx.value, ty.value

    def pixel_hits(self, dscene: DeviceScene, cam: Camera, y0: int, y1: int, max_hits: int = 64):
        c = cam.to_c()
        q = (y1 - y0) * cam.width
        hits = np.full(q * max_hits, -1, np.int32)
        counts = np.zeros(q, np.int32)
        self._check(self.lib.nx_debug_pixel_hits(self.ctx, dscene.handle, C.byref(c), y0, y1, max_hits,
                                                 hits.ctypes.data_as(_abi.PI32), counts.ctypes.data_as(_abi.PI32)))
        return hits.reshape(q, max_hits), counts

    def close(self):
        if self.ctx:
            self.lib.nx_ctx_destroy(self.ctx)
            self.ctx = None


# ---------------------------------------------------------------- reference-style value API
_default: dict = {}


class Optimizer:
    """The trainer's Adam over the 11 parameter groups (adam.cpp:9-42, trainer.cpp:238-323)
    on a device scene: fp64 moments, fp64 masters of the fp32-stored groups. Groups are
    numbered like ParamGroup (trainer.hpp:64-77): position, quat, scale, opacity, gamma,
    sh_dc, sh_rest, grid, w1, w2, w3."""
    GROUPS = ("position", "quat", "scale", "opacity", "gamma", "sh_dc", "sh_rest", "grid", "w1", "w2", "w3")

    def __init__(self, renderer: Renderer, dscene: DeviceScene):
        self.r, self.ds = renderer, dscene
        self.handle = C.c_void_p()
        renderer._check(renderer.lib.nx_optimizer_create(renderer.ctx, dscene.handle, C.byref(self.handle)))

    def step(self, grads_device: Sequence[int], configs: Sequence[Sequence[float]], stream: int = 0):
        """One adam_step per group from device SceneGrads pointers (prims, table, w1, w2,
        w3); configs: 11 (lr, beta1, beta2, eps); lr < 0 skips a group."""
        g = _abi.nx_grads(*grads_device)
        cfg = (_abi.nx_adam_config * _abi.NX_NUM_GROUPS)(*[_abi.nx_adam_config(*c) for c in configs])
        self.r._check(self.r.lib.nx_optimizer_step(self.r.ctx, self.handle, self.ds.handle, C.byref(g), cfg,
                                                   C.c_void_p(stream) if stream else None))

    def steps(self):
        out = (C.c_int64 * _abi.NX_NUM_GROUPS)()
        self.r._check(self.r.lib.nx_optimizer_steps(self.handle, out))
        return list(out)

    def size(self, group: int) -> int:
        n = C.c_int64()
        self.r._check(self.r.lib.nx_optimizer_size(self.handle, group, C.byref(n)))
        return n.value

    def set_params(self, group: int, values: np.ndarray):
        """Exact fp64 values of a group in its row layout (e.g. the unrounded initialisation)."""
        v = np.ascontiguousarray(values, np.float64).reshape(-1)
        self.r._check(self.r.lib.nx_optimizer_set_params(self.r.ctx, self.handle, self.ds.handle, group, _dp(v),
                                                         v.size))

    def download(self, group: int):
        """(params, m, v) of a group as float64 arrays."""
        n = self.size(group)
        p, m, v = np.zeros(n), np.zeros(n), np.zeros(n)
        self.r._check(self.r.lib.nx_optimizer_download(self.r.ctx, self.handle, self.ds.handle, group, _dp(p), _dp(m),
                                                       _dp(v)))
        return p, m, v

    def close(self):
        if self.handle:
            self.r.lib.nx_optimizer_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 — interpreter shutdown
            pass


def _renderer(device: int = 0) -> Renderer:
    r = _default.get(device)
    if r is None:
        r = _default[device] = Renderer(device)
    return r


def _device_scene(r: Renderer, scene: Scene) -> DeviceScene:
    key = scene.fingerprint()
    cache = _default.setdefault(("scenes", r.device), {})
    ds = cache.get(key)
    if ds is None:
        cache.clear()
        ds = cache[key] = r.upload(scene)
    ds.set_settings(scene.settings)
    return ds


def _value_frame(r: Renderer, device: int) -> DeviceFrame:
    fr = _default.get(("frame", device))
    if fr is None:
        fr = _default[("frame", device)] = r.frame()
        fr.set_backward(True)  # render_backward needs the fp64 base of the forward
    return fr


def _to_host_fb(fb: FrameBuffers) -> FrameBuffers:
    """Device-native dtypes -> the reference's fp64 FrameBuffers."""
    return FrameBuffers(fb.width, fb.height, fb.top_k, fb.base.astype(np.float64), fb.ids.copy(),
                        fb.depths.astype(np.float64), fb.weights.astype(np.float64), fb.texture.astype(np.float64),
                        fb.final_img.astype(np.float64), fb.residual.astype(np.float64))


def collection_pass(scene: Scene, cam: Camera, out: RenderResult, device: int = 0) -> None:
    """collection_pass (renderer.hpp:22): fills base/ids/depths/weights/residual."""
    r = _renderer(device)
    ds = _device_scene(r, scene)
    fr = _value_frame(r, device)
    r.collection_pass(ds, cam, fr)
    fb = _to_host_fb(fr.download(["base", "ids", "depths", "weights", "residual"]))
    fb.base = fr.base_f64()
    npix = cam.width * cam.height
    fb.texture = np.zeros(npix * scene.settings.top_k * 3)
    fb.final_img = np.zeros(npix * 3)
    out.fb = fb
    out.blended_error = np.zeros(scene.nexels.shape[0])


def texturing_pass(scene: Scene, cam: Camera, fb: FrameBuffers, device: int = 0) -> None:
    """texturing_pass (renderer.hpp:26): consumes fb's ids/depths/weights/base."""
    r = _renderer(device)
    ds = _device_scene(r, scene)
    fr = _value_frame(r, device)
    v = fr.view()
    if (v.width, v.height, v.top_k) != (fb.width, fb.height, fb.top_k):
        raise NexelError("invalid-argument", "FrameBuffers do not come from collection_pass on this camera")
    r.texturing_pass(ds, cam, fr)
    d = fr.download(["texture", "final_img"])
    fb.texture = d.texture.astype(np.float64)
    fb.final_img = d.final_img.astype(np.float64)


def render(scene: Scene, cam: Camera, device: int = 0) -> RenderResult:
    """render (renderer.hpp:28) = collection_pass + texturing_pass."""
    r = _renderer(device)
    ds = _device_scene(r, scene)
    fr = _value_frame(r, device)
    r.render(ds, cam, fr)
    fb = _to_host_fb(fr.download())
    fb.base = fr.base_f64()  # the reference's base is fp64; the device kept it for the reverse pass
    return RenderResult(fb, np.zeros(scene.nexels.shape[0]))


def render_backward(scene: Scene, cam: Camera, fb: FrameBuffers, up: UpstreamGrads, grads: SceneGrads,
                    err_pixel: Optional[np.ndarray] = None, blended_error: Optional[np.ndarray] = None,
                    device: int = 0) -> None:
    """render_backward (renderer.hpp:50-53): ``fb`` is the unmodified output of
    ``render(scene, cam)``; accumulates into ``grads`` (and into ``blended_error``
    when ``err_pixel`` is given). Top-K membership is treated as constant."""
    r = _renderer(device)
    ds = _device_scene(r, scene)
    fr = _value_frame(r, device)
    fr.upload(fb)
    r.render_backward(ds, cam, fr, up, grads, err_pixel, blended_error)


def losses_backward(scene: Scene, fb: FrameBuffers, gt: np.ndarray, w: LossWeights, grads: SceneGrads,
                    device: int = 0):
    """losses_backward (losses.hpp:52-56): returns (LossTerms as a dict, d_final,
    d_weights, d_texture) and accumulates the opacity / grid regularisers into ``grads``."""
    r = _renderer(device)
    ds = _device_scene(r, scene)
    fr = _value_frame(r, device)
    fr.upload(fb)
    return r.losses_backward(ds, fr, gt, w, grads)


# ---------------------------------------------------------------- synthetic inputs
def _synth(lib):
    """The generator's entry points (nx_synth.cpp) on `lib`: the product library by
    default, or the reference build in oracle/_ref, which links the same generator so
    that bench.py's reference arm never loads libnexel_b200.so."""
    if lib is None:
        return _abi.load()
    lib.nx_synth_stump_like.restype = C.c_int
    lib.nx_synth_stump_like.argtypes = [C.c_int64, C.c_double, C.c_uint64, C.c_double, C.c_int32, C.c_double,
                                        C.c_uint64, _abi.PD, C.POINTER(_abi.nx_settings),
                                        C.POINTER(_abi.nx_field_desc), _abi.PD, _abi.PD, _abi.PD, _abi.PD]
    lib.nx_synth_ring_camera.restype = C.c_int
    lib.nx_synth_ring_camera.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_abi.nx_camera)]
    return lib


def stump_like(n: int, coverage: float = 1.0, seed: int = 2512, ground_radius: float = 4.0,
               log2_table: int = 20, grid_init: float = 1e-4, field_seed: int = 2513, lib=None) -> Scene:
    lib = _synth(lib)
    s = _abi.nx_settings()
    d = _abi.nx_field_desc()
    nex = np.empty((n, 60), np.float64)
    lib.nx_synth_stump_like(n, coverage, seed, ground_radius, log2_table, grid_init, field_seed, None, None,
                            C.byref(d), None, None, None, None)
    nin = d.levels * d.features
    table = np.empty(d.levels * (1 << d.log2_table) * d.features, np.float64)
    w1 = np.empty(d.n_hidden * nin, np.float64)
    w2 = np.empty(d.n_hidden * d.n_hidden, np.float64)
    w3 = np.empty(48 * d.n_hidden, np.float64)
    st = lib.nx_synth_stump_like(n, coverage, seed, ground_radius, log2_table, grid_init, field_seed, _dp(nex),
                                 C.byref(s), C.byref(d), _dp(table), _dp(w1), _dp(w2), _dp(w3))
    if st != _abi.NX_OK:
        raise NexelError("invalid-argument", "stump_like: bad arguments")
    grid = HashGridConfig(d.levels, d.log2_table, d.features, d.base_scale, d.growth)
    return Scene(nex, TextureField(grid, table, w1, w2, w3, d.n_hidden), RenderSettings.from_c(s), extent=8.0)


def band_camera(cam: Camera, y0: int, rows: int) -> Camera:
    """Rows [y0, y0 + rows) of ``cam`` as a camera of its own (principal point shifted):
    every pixel keeps its ray (camera.hpp:32-35), hence its contributor list and
    colour — the image-band sharding of SURVEY.md §8(e) needs no collective."""
    if y0 < 0 or rows < 0 or y0 + rows > cam.height:
        raise NexelError("invalid-argument", "band outside the image")
    return Camera(cam.width, rows, cam.fx, cam.fy, cam.cx, cam.cy - y0, cam.R, cam.t, f"{cam.name}[{y0}:{y0 + rows}]")


def image_bands(height: int, n: int, align: int = 16):
    """n contiguous row bands covering the image, tile-aligned (the last one shorter)."""
    step = -(-height // n)
    step = -(-step // align) * align
    out = []
    for i in range(n):
        y0 = min(i * step, height)
        out.append((y0, max(0, min(height, y0 + step) - y0)))
    return out


def ring_camera(index: int, n_views: int = 256, width: int = 1920, height: int = 1080, lib=None) -> Camera:
    lib = _synth(lib)
    c = _abi.nx_camera()
    st = lib.nx_synth_ring_camera(index, n_views, width, height, C.byref(c))
    if st != _abi.NX_OK:
        raise NexelError("invalid-argument", "ring_camera: bad arguments")
    return Camera.from_c(c, name=f"ring{index}")
