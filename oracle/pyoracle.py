"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes bindings of the two CPU checkers of the render path:

* ``Oracle``    — oracle/build/libnexel_oracle.so, the plain-C restatement
                  (oracle/nexel_oracle.c), scalar single-thread fp64;
* ``Reference`` — oracle/_ref/libnexel_ref_{v4,v3}.so, the reference's own
                  render path compiled in place from /root/reference by
                  oracle/Makefile (multi-threaded via NEXEL_THREADS).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg use this.
Both take the data containers of paper_2512_13796_b200.api (Scene, Camera).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2512_13796_b200 import _abi
from paper_2512_13796_b200.api import Camera, HashGridConfig, RenderSettings, Scene, TextureField

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "build", "libnexel_oracle.so")
REF_DIR = os.path.join(HERE, "_ref")

PD, PI32, PI64 = _abi.PD, _abi.PI32, _abi.PI64
P = C.c_void_p


class OracleError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.code = _abi.STATUS_CODES.get(status, "error")


def _dp(a):
    return None if a is None else a.ctypes.data_as(PD)


def _scene_args(scene: Scene):
    nex = np.ascontiguousarray(scene.nexels, dtype=np.float64).reshape(-1, 60)
    f = scene.field
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (f.table, f.w1, f.w2, f.w3)]
    return nex, f.desc(), arrs


class FB:
    """fp64 FrameBuffers as produced by the CPU checkers."""

    def __init__(self, W, H, K):
        n = W * H
        self.width, self.height, self.top_k = W, H, K
        self.base = np.zeros(n * 3)
        self.ids = np.full(n * K, -1, np.int32)
        self.depths = np.zeros(n * K)
        self.weights = np.zeros(n * K)
        self.texture = np.zeros(n * K * 3)
        self.final_img = np.zeros(n * 3)
        self.residual = np.ones(n)


class _Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n_entries", "n_straddlers", "tile_keys", "n_queries", "n_tests", "n_hits")]


class Oracle:
    """Plain-C restatement (oracle/nexel_oracle.c)."""

    def __init__(self, path: str = ORACLE_LIB):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C oracle oracle`")
        L = self.lib = C.CDLL(path)
        S = C.POINTER(_abi.nx_settings)
        F = C.POINTER(_abi.nx_field_desc)
        Cm = C.POINTER(_abi.nx_camera)
        L.orc_last_error.restype = C.c_char_p
        L.orc_render.argtypes = [S, C.c_int64, PD, F, PD, PD, PD, PD, Cm, PD, PI32, PD, PD, PD, PD, PD,
                                 C.POINTER(_Stats)]
        L.orc_tile_lists.argtypes = [S, C.c_int64, PD, Cm, PI64, PI32, C.c_int64, PI64, PI32, PI32]
        L.orc_pixel_hits.argtypes = [S, C.c_int64, PD, Cm, C.c_int, C.c_int, C.c_int, PI32, PI32]
        for name in ("orc_eval_kernel",):
            getattr(L, name).restype = C.c_double
            getattr(L, name).argtypes = [C.c_double] * 5
        L.orc_support_radius.restype = C.c_double
        L.orc_support_radius.argtypes = [C.c_double, C.c_double]
        L.orc_hash_cell.restype = C.c_uint32
        L.orc_hash_cell.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint32]
        L.orc_map_positive.restype = C.c_uint64
        L.orc_map_positive.argtypes = [C.c_int64]
        L.orc_downweight.restype = C.c_double
        L.orc_downweight.argtypes = [C.c_double] * 3
        L.orc_sh_basis.argtypes = [PD, PD]
        L.orc_topk.argtypes = [C.c_int, C.c_int, PI32, PD, PD, PI32, PD]
        L.orc_field_forward.argtypes = [F, PD, PD, PD, PD, C.c_int64, PD, C.c_int, PD]

    def _check(self, st):
        if st:
            raise OracleError(st, self.lib.orc_last_error().decode())

    def render(self, scene: Scene, cam: Camera):
        nex, d, (tab, w1, w2, w3) = _scene_args(scene)
        s = scene.settings.to_c()
        c = cam.to_c()
        fb = FB(cam.width, cam.height, scene.settings.top_k)
        st = _Stats()
        self._check(self.lib.orc_render(C.byref(s), nex.shape[0], _dp(nex), C.byref(d), _dp(tab), _dp(w1), _dp(w2),
                                        _dp(w3), C.byref(c), _dp(fb.base), fb.ids.ctypes.data_as(PI32),
                                        _dp(fb.depths), _dp(fb.weights), _dp(fb.texture), _dp(fb.final_img),
                                        _dp(fb.residual), C.byref(st)))
        fb.stats = {k: int(getattr(st, k)) for k, _ in _Stats._fields_}
        return fb

    def tile_lists(self, scene: Scene, cam: Camera):
        nex = np.ascontiguousarray(scene.nexels, dtype=np.float64).reshape(-1, 60)
        s, c = scene.settings.to_c(), cam.to_c()
        total, tx, ty = C.c_int64(), C.c_int32(), C.c_int32()
        self._check(self.lib.orc_tile_lists(C.byref(s), nex.shape[0], _dp(nex), C.byref(c), None, None, 0,
                                            C.byref(total), C.byref(tx), C.byref(ty)))
        off = np.empty(tx.value * ty.value + 1, np.int64)
        ids = np.empty(max(total.value, 1), np.int32)
        self._check(self.lib.orc_tile_lists(C.byref(s), nex.shape[0], _dp(nex), C.byref(c),
                                            off.ctypes.data_as(PI64), ids.ctypes.data_as(PI32), total.value,
                                            C.byref(total), C.byref(tx), C.byref(ty)))
        return off, ids[: total.value], tx.value, ty.value

    def pixel_hits(self, scene: Scene, cam: Camera, y0: int, y1: int, max_hits: int = 64):
        nex = np.ascontiguousarray(scene.nexels, dtype=np.float64).reshape(-1, 60)
        s, c = scene.settings.to_c(), cam.to_c()
        q = (y1 - y0) * cam.width
        hits = np.full(q * max_hits, -1, np.int32)
        counts = np.zeros(q, np.int32)
        self._check(self.lib.orc_pixel_hits(C.byref(s), nex.shape[0], _dp(nex), C.byref(c), y0, y1, max_hits,
                                            hits.ctypes.data_as(PI32), counts.ctypes.data_as(PI32)))
        return hits.reshape(q, max_hits), counts

    def field_forward(self, field: TextureField, queries: np.ndarray, no_downweight=False):
        q = np.ascontiguousarray(queries, dtype=np.float64).reshape(-1, 8)
        out = np.empty((q.shape[0], 3))
        d = field.desc()
        arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (field.table, field.w1, field.w2, field.w3)]
        self._check(self.lib.orc_field_forward(C.byref(d), *[_dp(a) for a in arrs], q.shape[0], _dp(q),
                                               int(no_downweight), _dp(out)))
        return out


def _cpu_flags() -> set:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def reference_lib_path() -> str | None:
    """The in-place build of the reference for this host's ISA (x86-64-v4 if AVX-512)."""
    v4 = os.path.join(REF_DIR, "libnexel_ref_v4.so")
    v3 = os.path.join(REF_DIR, "libnexel_ref_v3.so")
    flags = _cpu_flags()
    if os.path.exists(v4) and {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= flags:
        return v4
    return v3 if os.path.exists(v3) else None


class Reference:
    """The reference's own render path (compiled in place from /root/reference)."""

    def stump_like(self, n: int, **kw) -> Scene:
        """The synthetic scene from the generator linked into this
        library: the reference arm builds its inputs without the product library."""
        from paper_2512_13796_b200.api import stump_like
        return stump_like(n, lib=self.lib, **kw)

    def ring_camera(self, index: int, n_views: int = 256, width: int = 1920, height: int = 1080) -> Camera:
        from paper_2512_13796_b200.api import ring_camera
        return ring_camera(index, n_views, width, height, lib=self.lib)

    def __init__(self, path: str | None = None):
        path = path or reference_lib_path()
        if not path or not os.path.exists(path):
            raise ImportError("oracle/_ref not built (needs /root/reference at build time)")
        self.path = path
        L = self.lib = C.CDLL(path)
        S = C.POINTER(_abi.nx_settings)
        F = C.POINTER(_abi.nx_field_desc)
        Cm = C.POINTER(_abi.nx_camera)
        L.ref_last_error.restype = C.c_char_p
        L.ref_scene_create.argtypes = [S, C.c_int64, PD, F, PD, PD, PD, PD, C.POINTER(P)]
        L.ref_scene_destroy.argtypes = [P]
        L.ref_scene_set_settings.argtypes = [P, S]
        L.ref_render.argtypes = [P, Cm, PD, PI32, PD, PD, PD, PD, PD]
        L.ref_naive_render.argtypes = [P, Cm, PD]
        L.ref_tile_lists.argtypes = [P, Cm, PI64, PI32, C.c_int64, PI64, PI32, PI32]
        L.ref_pixel_hits.argtypes = [P, Cm, C.c_int, C.c_int, C.c_int, PI32, PI32]
        L.ref_gen_random_scene.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                           C.c_double, C.c_int, C.c_int, C.c_double, C.c_double, PD, S, F, PD, PD,
                                           PD, PD, Cm]
        L.ref_gen_field.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_int, F, PD, PD, PD, PD]
        L.ref_gen_field_for_extent.argtypes = [C.c_uint64, C.c_double, C.c_int, C.c_int, C.c_double, F, PD, PD, PD,
                                               PD]
        L.ref_look_at_camera.argtypes = [PD, PD, C.c_int, C.c_double, Cm]
        L.ref_eval_kernel.restype = C.c_double
        L.ref_eval_kernel.argtypes = [C.c_double] * 5
        L.ref_support_radius.restype = C.c_double
        L.ref_support_radius.argtypes = [C.c_double] * 2
        L.ref_hash_cell.restype = C.c_uint32
        L.ref_hash_cell.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint32]
        L.ref_downweight.restype = C.c_double
        L.ref_downweight.argtypes = [C.c_double] * 3
        L.ref_field_forward.argtypes = [P, C.c_int64, PD, C.c_int, PD]
        L.ref_render_backward.argtypes = [P, Cm, PD, PD, PD, PD, PD, PD, PD, PD, PD, PD]
        L.ref_save_checkpoint.argtypes = [P, C.c_char_p, Cm, C.c_int, C.c_uint64, C.c_double]
        L.ref_adam_step.argtypes = [PD, PD, PI64, PD, PD, PD, C.c_int64]
        L.ref_densify_split.argtypes = [PD, C.c_int64, C.c_int64, PD, C.c_int64, C.c_double, C.c_uint64, PD, PI32,
                                        PI64, PI64]
        L.ref_prune.argtypes = [PD, C.c_int64, C.c_double, PI32, PI64]
        L.ref_adam_remap_rows.argtypes = [PD, PD, C.c_int64, C.c_int64, PI32, C.c_int64]
        L.ref_losses_backward.argtypes = [P, C.c_int, C.c_int, C.c_int, PI32, PD, PD, PD, PD, PD, PD, PD, PD, PD,
                                          PD, PD]
        self._scene = None
        self._scene_key = None

    def _check(self, st):
        if st:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def _handle(self, scene: Scene):
        key = scene.fingerprint()  # content-keyed: ids / buffers of freed scenes get reused
        if self._scene is None or self._scene_key != key:
            self.close()
            nex, d, (tab, w1, w2, w3) = _scene_args(scene)
            s = scene.settings.to_c()
            h = P()
            self._check(self.lib.ref_scene_create(C.byref(s), nex.shape[0], _dp(nex), C.byref(d), _dp(tab), _dp(w1),
                                                  _dp(w2), _dp(w3), C.byref(h)))
            self._scene, self._scene_key = h, key
        s = scene.settings.to_c()
        self.lib.ref_scene_set_settings(self._scene, C.byref(s))
        return self._scene

    def close(self):
        if self._scene:
            self.lib.ref_scene_destroy(self._scene)
            self._scene = None

    def render(self, scene: Scene, cam: Camera):
        h = self._handle(scene)
        fb = FB(cam.width, cam.height, scene.settings.top_k)
        c = cam.to_c()
        self._check(self.lib.ref_render(h, C.byref(c), _dp(fb.base), fb.ids.ctypes.data_as(PI32), _dp(fb.depths),
                                        _dp(fb.weights), _dp(fb.texture), _dp(fb.final_img), _dp(fb.residual)))
        return fb

    def naive_render(self, scene: Scene, cam: Camera):
        h = self._handle(scene)
        img = np.zeros(cam.width * cam.height * 3)
        c = cam.to_c()
        self._check(self.lib.ref_naive_render(h, C.byref(c), _dp(img)))
        return img

    def tile_lists(self, scene: Scene, cam: Camera):
        h = self._handle(scene)
        c = cam.to_c()
        total, tx, ty = C.c_int64(), C.c_int32(), C.c_int32()
        self._check(self.lib.ref_tile_lists(h, C.byref(c), None, None, 0, C.byref(total), C.byref(tx), C.byref(ty)))
        off = np.empty(tx.value * ty.value + 1, np.int64)
        ids = np.empty(max(total.value, 1), np.int32)
        self._check(self.lib.ref_tile_lists(h, C.byref(c), off.ctypes.data_as(PI64), ids.ctypes.data_as(PI32),
                                            total.value, C.byref(total), C.byref(tx), C.byref(ty)))
        return off, ids[: total.value], tx.value, ty.value

    def pixel_hits(self, scene: Scene, cam: Camera, y0: int, y1: int, max_hits: int = 64):
        h = self._handle(scene)
        c = cam.to_c()
        q = (y1 - y0) * cam.width
        hits = np.full(q * max_hits, -1, np.int32)
        counts = np.zeros(q, np.int32)
        self._check(self.lib.ref_pixel_hits(h, C.byref(c), y0, y1, max_hits, hits.ctypes.data_as(PI32),
                                            counts.ctypes.data_as(PI32)))
        return hits.reshape(q, max_hits), counts

    def field_forward(self, scene: Scene, queries: np.ndarray, no_downweight=False):
        h = self._handle(scene)
        q = np.ascontiguousarray(queries, dtype=np.float64).reshape(-1, 8)
        out = np.empty((q.shape[0], 3))
        self._check(self.lib.ref_field_forward(h, q.shape[0], _dp(q), int(no_downweight), _dp(out)))
        return out

    def render_backward(self, scene: Scene, cam: Camera, d_final=None, d_weights=None, d_texture=None,
                        err_pixel=None):
        """render + render_backward of the reference (renderer.cpp:239-401) with the
        given upstream gradients; returns (prims (N,60), table, w1, w2, w3, blended_error)."""
        h = self._handle(scene)
        c = cam.to_c()
        f = scene.field
        g = [np.zeros((scene.nexels.shape[0], 60)), np.zeros(f.grid.param_count()), np.zeros(np.size(f.w1)),
             np.zeros(np.size(f.w2)), np.zeros(np.size(f.w3))]
        be = np.zeros(scene.nexels.shape[0]) if err_pixel is not None else None

        def opt(a):
            return None if a is None else _dp(np.ascontiguousarray(a, np.float64))
        keep = [np.ascontiguousarray(a, np.float64) if a is not None else None
                for a in (d_final, d_weights, d_texture, err_pixel)]
        self._check(self.lib.ref_render_backward(h, C.byref(c), *(opt(a) for a in keep), *(_dp(a) for a in g),
                                                 _dp(be) if be is not None else None))
        return (*g, be)

    def losses_backward(self, scene: Scene, W: int, H: int, K: int, ids, weights, texture, final_img, gt, lw,
                        g_prims=None, g_table=None):
        """losses_backward of the reference (losses.cpp:107-238) on the given buffers;
        returns (terms dict, d_final, d_weights, d_texture, g_prims, g_table)."""
        h = self._handle(scene)
        npix = W * H
        ids = np.ascontiguousarray(ids, np.int32)
        arr = [np.ascontiguousarray(a, np.float64) for a in (weights, texture, final_img, gt, lw)]
        d_final, d_weights, d_texture = np.zeros(npix * 3), np.zeros(max(npix * K, 1)), np.zeros(max(npix * K * 3, 1))
        gp = np.zeros((scene.nexels.shape[0], 60)) if g_prims is None else np.array(g_prims, np.float64)
        gtab = np.zeros(scene.field.grid.param_count()) if g_table is None else np.array(g_table, np.float64)
        terms = np.zeros(8)
        self._check(self.lib.ref_losses_backward(h, W, H, K, ids.ctypes.data_as(PI32), *(_dp(a) for a in arr),
                                                 _dp(d_final), _dp(d_weights), _dp(d_texture), _dp(gp), _dp(gtab),
                                                 _dp(terms)))
        keys = ("l1", "dssim", "image", "texture", "alpha", "opacity", "grid", "total")
        return dict(zip(keys, terms.tolist())), d_final, d_weights[: npix * K], d_texture[: npix * K * 3], gp, gtab

    def save_checkpoint(self, scene: Scene, path: str, cams, iteration: int = 0):
        """save_checkpoint (checkpoint.cpp:99-171) of the scene with the cameras."""
        h = self._handle(scene)
        arr = (_abi.nx_camera * max(len(cams), 1))(*[c.to_c() for c in cams])
        self._check(self.lib.ref_save_checkpoint(h, str(path).encode(), arr, len(cams), iteration, scene.extent))

    def adam_step(self, m, v, step: int, cfg, params, grads):
        """adam_step (adam.cpp:9-22): updates params, m, v in place; returns the new step."""
        st = C.c_int64(step)
        c = np.ascontiguousarray(cfg, np.float64)
        self._check(self.lib.ref_adam_step(_dp(m), _dp(v), C.byref(st), _dp(c), _dp(params),
                                           _dp(np.ascontiguousarray(grads, np.float64)), params.size))
        return st.value

    def densify_split(self, nexels, errors, budget: int, split_fraction: float, seed: int):
        """densify_split (density.cpp:102-161) with mt19937_64(seed): returns (nexels,
        new_to_old, split_count, uniforms consumed)."""
        n = nexels.shape[0]
        cap = n + int(np.ceil(split_fraction * n)) + 1
        buf = np.zeros((cap, 60))
        buf[:n] = nexels
        u = np.zeros(n)
        n2o = np.zeros(cap, np.int32)
        n_out, sc = C.c_int64(), C.c_int64()
        self._check(self.lib.ref_densify_split(_dp(buf), n, cap, _dp(np.ascontiguousarray(errors, np.float64)),
                                               budget, split_fraction, seed, _dp(u), n2o.ctypes.data_as(PI32),
                                               C.byref(n_out), C.byref(sc)))
        return buf[: n_out.value], n2o[: n_out.value], sc.value, u

    def prune(self, nexels, min_opacity: float):
        n = nexels.shape[0]
        buf = np.ascontiguousarray(nexels, np.float64).copy()
        n2o = np.zeros(max(n, 1), np.int32)
        n_out = C.c_int64()
        self._check(self.lib.ref_prune(_dp(buf), n, min_opacity, n2o.ctypes.data_as(PI32), C.byref(n_out)))
        return buf[: n_out.value], n2o[: n_out.value]

    def adam_remap_rows(self, m, v, new_to_old, width: int):
        """adam_remap_rows (adam.cpp:24-42): returns the remapped (m, v)."""
        rows_new = len(new_to_old)
        m2 = np.zeros(max(m.size, rows_new * width))
        v2 = np.zeros(max(v.size, rows_new * width))
        m2[: m.size] = m
        v2[: v.size] = v
        n2o = np.ascontiguousarray(new_to_old, np.int32)
        self._check(self.lib.ref_adam_remap_rows(_dp(m2), _dp(v2), m.size // width, rows_new,
                                                 n2o.ctypes.data_as(PI32), width))
        return m2[: rows_new * width].copy(), v2[: rows_new * width].copy()

    # ---- the reference test generators (tests/helpers.hpp:88-125)
    def random_scene(self, seed: int, n_prims: int, top_k: int, res: int, focal: float, dist: float,
                     op_lo: float = 0.35, op_hi: float = 0.85, levels: int = 4, log2_table: int = 5,
                     grid_init: float = 1e-2, hidden: int = 16):
        nin = levels * 2
        nex = np.zeros((n_prims, 60))
        tab = np.zeros(levels * (1 << log2_table) * 2)
        w1, w2, w3 = np.zeros(hidden * nin), np.zeros(hidden * hidden), np.zeros(48 * hidden)
        s, d, c = _abi.nx_settings(), _abi.nx_field_desc(), _abi.nx_camera()
        self._check(self.lib.ref_gen_random_scene(seed, n_prims, top_k, op_lo, op_hi, levels, log2_table, grid_init,
                                                  hidden, res, focal, dist, _dp(nex), C.byref(s), C.byref(d),
                                                  _dp(tab), _dp(w1), _dp(w2), _dp(w3), C.byref(c)))
        grid = HashGridConfig(d.levels, d.log2_table, d.features, d.base_scale, d.growth)
        scene = Scene(nex, TextureField(grid, tab, w1, w2, w3, d.n_hidden), RenderSettings.from_c(s))
        return scene, Camera.from_c(c, "test")

    def field(self, seed: int, levels: int, log2_table: int, grid_init: float, hidden: int) -> TextureField:
        nin = levels * 2
        tab = np.zeros(levels * (1 << log2_table) * 2)
        w1, w2, w3 = np.zeros(hidden * nin), np.zeros(hidden * hidden), np.zeros(48 * hidden)
        d = _abi.nx_field_desc()
        self._check(self.lib.ref_gen_field(seed, levels, log2_table, grid_init, hidden, C.byref(d), _dp(tab), _dp(w1),
                                           _dp(w2), _dp(w3)))
        grid = HashGridConfig(d.levels, d.log2_table, d.features, d.base_scale, d.growth)
        return TextureField(grid, tab, w1, w2, w3, d.n_hidden)

    def field_for_extent(self, seed: int, extent: float, levels: int, log2_table: int,
                         grid_init: float) -> TextureField:
        nin = levels * 2
        tab = np.zeros(levels * (1 << log2_table) * 2)
        w1, w2, w3 = np.zeros(64 * nin), np.zeros(64 * 64), np.zeros(48 * 64)
        d = _abi.nx_field_desc()
        self._check(self.lib.ref_gen_field_for_extent(seed, extent, levels, log2_table, grid_init, C.byref(d),
                                                      _dp(tab), _dp(w1), _dp(w2), _dp(w3)))
        grid = HashGridConfig(d.levels, d.log2_table, d.features, d.base_scale, d.growth)
        return TextureField(grid, tab, w1, w2, w3, d.n_hidden)

    def look_at(self, pos, target, res: int, focal: float) -> Camera:
        c = _abi.nx_camera()
        p = np.asarray(pos, np.float64)
        t = np.asarray(target, np.float64)
        self._check(self.lib.ref_look_at_camera(_dp(p), _dp(t), res, focal, C.byref(c)))
        return Camera.from_c(c, "test")
