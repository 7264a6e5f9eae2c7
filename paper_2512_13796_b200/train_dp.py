"""Data-parallel training iteration over views (BASELINE config 5 on
N GPUs): one process per GPU, each holding a replica of the scene and the optimizer
state; per iteration every rank renders its own view (trainer.cpp:274), runs
losses_backward (:281), the per-pixel error map (:288-296) and render_backward
(:299), the ranks average their gradients (and sum their blended-error maps, which
drive density control, :301-302) with one all-reduce per array, and every rank applies
the same Adam step (:305-323) — so the replicas stay bit-identical.

The all-reduce runs over torch.distributed: NCCL on the device arrays (NVLink /
NVSwitch) when the process group is NCCL, or through host copies for gloo (the CPU
backend the tests use to run two ranks on one GPU).
"""
import ctypes as C
from typing import List, Optional

import numpy as np

from . import _abi

# Adam groups with the trainer's default rates (trainer.hpp:30-42, trainer.cpp:238-250);
# group 0's rate scales with the scene extent.
DEFAULT_RATES = [(1.6e-4, 1e-15), (1e-3, 1e-8), (5e-3, 1e-8), (5e-2, 1e-8), (2e-3, 1e-8), (2.5e-3, 1e-8),
                 (1.25e-4, 1e-8), (1e-2, 1e-8), (1e-3, 1e-8), (1e-3, 1e-8), (1e-3, 1e-8)]


def device_view(ptr: int, n: int, dtype, device):
    """A torch view of a device array owned by the library (no copy)."""
    import torch

    class _CAI:
        def __init__(self):
            typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4"}[dtype]
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False),
                                             "version": 3}
    return torch.as_tensor(_CAI(), device=device)


def rank_views(n_views: int, n_iters: int, world: int, rank: int, seed: int = 3) -> List[int]:
    """The view of each iteration for this rank: one permutation of the training views
    per epoch (trainer.cpp:266-272 shuffles per epoch), dealt to the ranks in turn
    (iteration i, rank r takes position i * world + r of the epoch stream)."""
    rng = np.random.default_rng(seed)
    order: List[int] = []
    while len(order) < n_iters * world:
        order.extend(int(v) for v in rng.permutation(n_views))
    return [order[i * world + rank] for i in range(n_iters)]


class DataParallelStep:
    """One training iteration of a device scene on this rank's view, gradients averaged
    across ``dist`` (None: one process). ``gt`` maps a view index to its fp64 ground
    truth on the device (torch tensor, H*W*3)."""

    def __init__(self, renderer, dscene, scene, cams, gt, dist=None, stream=None, rates=DEFAULT_RATES):
        import torch
        self.r, self.ds, self.cams, self.gt, self.dist = renderer, dscene, cams, gt, dist
        self.dev = torch.device("cuda", renderer.device)
        self.stream = stream if stream is not None else torch.cuda.ExternalStream(renderer.stream, device=self.dev)
        cam0 = next(iter(cams.values()))
        K = scene.settings.top_k
        npix = cam0.width * cam0.height
        f = scene.field
        z = lambda n: torch.zeros(n, dtype=torch.float64, device=self.dev)  # noqa: E731
        self.d_final, self.d_weights, self.d_texture, self.err = z(npix * 3), z(npix * K), z(npix * K * 3), z(npix)
        self.grads = [z(scene.nexels.shape[0] * _abi.NX_PARAMS_PER_NEXEL), z(f.grid.param_count()), z(f.w1.size),
                      z(f.w2.size), z(f.w3.size)]
        self.blend = z(scene.nexels.shape[0])       # blended error, accumulated over iterations
        self.blend_step = z(scene.nexels.shape[0])  # this iteration's share (all-reduced, then added)
        self.terms = z(8)
        self.up = _abi.nx_upstream(self.d_final.data_ptr(), self.d_weights.data_ptr(), self.d_texture.data_ptr())
        self.gg = _abi.nx_grads(*(t.data_ptr() for t in self.grads))
        self.lw = _abi.nx_loss_weights()
        renderer.lib.nx_loss_weights_default(C.byref(self.lw))
        cfg = [(lr * (scene.extent if g == 0 else 1.0), eps) for g, (lr, eps) in enumerate(rates)]
        self.acfg = (_abi.nx_adam_config * _abi.NX_NUM_GROUPS)(*[_abi.nx_adam_config(lr, 0.9, 0.999, eps)
                                                                 for lr, eps in cfg])
        self.opt = C.c_void_p()
        renderer._check(renderer.lib.nx_optimizer_create(renderer.ctx, dscene.handle, C.byref(self.opt)))
        self.frame = renderer.frame()
        self.frame.set_backward(True)
        self._nccl = dist is not None and dist.get_backend() == "nccl"

    def _all_reduce(self, tensors, average):
        import torch
        world = self.dist.get_world_size()
        for t in tensors:
            if self._nccl:
                with torch.cuda.stream(self.stream):
                    self.dist.all_reduce(t)
                    if average:
                        t.mul_(1.0 / world)
            else:  # gloo: through host copies
                torch.cuda.current_stream(self.dev).wait_stream(self.stream)
                h = t.cpu()
                self.dist.all_reduce(h)
                if average:
                    h.mul_(1.0 / world)
                with torch.cuda.stream(self.stream):
                    t.copy_(h)

    def step(self, view: int, reduce_blend: bool = True):
        """render -> losses_backward -> error map -> render_backward -> all-reduce ->
        Adam, all on the renderer's stream; returns the rank's loss terms (device)."""
        import torch
        r, lib, s = self.r, self.r.lib, C.c_void_p(self.r.stream)
        c = self.cams[view].to_c()
        gt = self.gt[view]
        with torch.cuda.stream(self.stream):  # SceneGrads::allocate every iteration (renderer.cpp:245-248)
            for t in self.grads:
                t.zero_()
            self.blend_step.zero_()
        r._check(lib.nx_render(r.ctx, self.ds.handle, C.byref(c), self.frame.handle, s))
        r._check(lib.nx_losses_backward(r.ctx, self.ds.handle, self.frame.handle, C.c_void_p(gt.data_ptr()),
                                        C.byref(self.lw), C.c_void_p(self.d_final.data_ptr()),
                                        C.c_void_p(self.d_weights.data_ptr()), C.c_void_p(self.d_texture.data_ptr()),
                                        C.byref(self.gg), C.c_void_p(self.terms.data_ptr()), s))
        r._check(lib.nx_pixel_error(r.ctx, self.frame.handle, C.c_void_p(gt.data_ptr()),
                                    C.c_void_p(self.err.data_ptr()), s))
        r._check(lib.nx_render_backward(r.ctx, self.ds.handle, C.byref(c), self.frame.handle, C.byref(self.up),
                                        C.byref(self.gg), C.c_void_p(self.err.data_ptr()),
                                        C.c_void_p(self.blend_step.data_ptr()), s))
        if self.dist is not None and self.dist.get_world_size() > 1:
            self._all_reduce(self.grads, average=True)
            if reduce_blend:
                self._all_reduce([self.blend_step], average=False)
        with torch.cuda.stream(self.stream):
            self.blend.add_(self.blend_step)
        r._check(lib.nx_optimizer_step(r.ctx, self.opt, self.ds.handle, C.byref(self.gg), self.acfg, s))
        return self.terms

    def close(self):
        self.frame.close()
        if self.opt:
            self.r.lib.nx_optimizer_destroy(self.opt)
            self.opt = C.c_void_p()
