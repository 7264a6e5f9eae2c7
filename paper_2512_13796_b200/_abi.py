"""ctypes mirror of include/nexel_b200.h and the loader of the in-tree library.

The product path is the CUDA library ``libnexel_b200.so`` built in-tree by
``__graft_entry__.build()`` / ``make lib``. There is no CPU fallback: if the
library is missing, ``load()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnexel_b200.so")

NX_OK = 0
NX_BAD_SETTINGS = 1
NX_BAD_CAMERA = 2
NX_BAD_PRIMITIVE = 3
NX_MISSING_FILE = 4
NX_BAD_CHECKPOINT = 5
NX_INVALID_ARGUMENT = 10
NX_UNSUPPORTED = 11
NX_OUT_OF_MEMORY = 12
NX_CUDA_ERROR = 13
NX_NO_DEVICE = 14

NX_MAX_TOP_K = 8
NX_PRECISION_DEFAULT = 0
NX_PRECISION_F64 = 1
NX_PARAMS_PER_NEXEL = 60
NX_SH_VALUES = 48
NX_NUM_STAGES = 7
STAGE_NAMES = ("preprocess", "depth_sort", "emit", "tile_sort", "composite", "texture", "texture_mlp")

STATUS_CODES = {
    NX_BAD_SETTINGS: "bad-settings",
    NX_BAD_CAMERA: "bad-camera",
    NX_BAD_PRIMITIVE: "bad-primitive",
    NX_MISSING_FILE: "missing-file",
    NX_BAD_CHECKPOINT: "bad-checkpoint",
    NX_INVALID_ARGUMENT: "invalid-argument",
    NX_UNSUPPORTED: "unsupported",
    NX_OUT_OF_MEMORY: "out-of-memory",
    NX_CUDA_ERROR: "cuda-error",
    NX_NO_DEVICE: "no-device",
}


class nx_settings(C.Structure):
    _fields_ = [
        ("top_k", C.c_int32),
        ("tile", C.c_int32),
        ("background", C.c_double * 3),
        ("near_eps", C.c_double),
        ("alpha_max", C.c_double),
        ("min_transmittance", C.c_double),
        ("no_gamma", C.c_int32),
        ("no_prim_sh", C.c_int32),
        ("no_downweight", C.c_int32),
        ("precision", C.c_int32),
    ]


class nx_field_desc(C.Structure):
    _fields_ = [
        ("levels", C.c_int32),
        ("log2_table", C.c_int32),
        ("features", C.c_int32),
        ("n_hidden", C.c_int32),
        ("base_scale", C.c_double),
        ("growth", C.c_double),
    ]


class nx_camera(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("fx", C.c_double),
        ("fy", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("R", C.c_double * 9),
        ("t", C.c_double * 3),
    ]


class nx_frame_view(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("top_k", C.c_int32),
        ("tiles_x", C.c_int32),
        ("tiles_y", C.c_int32),
        ("base", C.c_void_p),
        ("ids", C.c_void_p),
        ("depths", C.c_void_p),
        ("weights", C.c_void_p),
        ("texture", C.c_void_p),
        ("final_img", C.c_void_p),
        ("residual", C.c_void_p),
    ]


class nx_host_frame(C.Structure):
    _fields_ = [
        ("base", C.c_void_p),
        ("ids", C.c_void_p),
        ("depths", C.c_void_p),
        ("weights", C.c_void_p),
        ("texture", C.c_void_p),
        ("final_img", C.c_void_p),
        ("residual", C.c_void_p),
        ("base_f64", C.c_void_p),
        ("residual_f64", C.c_void_p),
        ("texture_f64", C.c_void_p),
        ("final_f64", C.c_void_p),
        ("weights_f32", C.c_void_p),
    ]


class nx_upstream(C.Structure):
    _fields_ = [
        ("d_final", C.c_void_p),
        ("d_weights", C.c_void_p),
        ("d_texture", C.c_void_p),
    ]


class nx_grads(C.Structure):
    _fields_ = [
        ("prims", C.c_void_p),
        ("table", C.c_void_p),
        ("w1", C.c_void_p),
        ("w2", C.c_void_p),
        ("w3", C.c_void_p),
    ]


class nx_loss_weights(C.Structure):
    _fields_ = [("dssim", C.c_double), ("alpha", C.c_double), ("texture", C.c_double), ("opacity", C.c_double),
                ("grid", C.c_double)]


class nx_loss_terms(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("l1", "dssim", "image", "texture", "alpha", "opacity", "grid", "total")]

    def as_dict(self):
        return {k: float(getattr(self, k)) for k, _ in self._fields_}


class nx_nexl_info(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("n_nexels", C.c_int64), ("n_cameras", C.c_int32),
                ("has_optimizer", C.c_int32), ("extent", C.c_double), ("settings", nx_settings),
                ("field", nx_field_desc)]


class nx_adam_config(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]


NX_NUM_GROUPS = 11
GROUP_NAMES = ("position", "quat", "scale", "opacity", "gamma", "sh_dc", "sh_rest", "grid", "w1", "w2", "w3")


class nx_frame_stats(C.Structure):
    _fields_ = [
        ("n_nexels", C.c_int64),
        ("n_entries", C.c_int64),
        ("n_dropped_support", C.c_int64),
        ("n_behind", C.c_int64),
        ("n_offscreen", C.c_int64),
        ("n_rect", C.c_int64),
        ("n_straddlers", C.c_int64),
        ("n_straddlers_kept", C.c_int64),
        ("tile_keys", C.c_int64),
        ("work_keys", C.c_int64),
        ("n_queries", C.c_int64),
        ("near_alpha", C.c_int64),
        ("near_transmittance", C.c_int64),
        ("near_topk", C.c_int64),
        ("near_depth", C.c_int64),
        ("near_rect", C.c_int64),
        ("near_support", C.c_int64),
        ("redo_tiles", C.c_int64),
    ]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
D = C.c_double
PD = C.POINTER(C.c_double)
PI32 = C.POINTER(C.c_int32)
PI64 = C.POINTER(C.c_int64)
PF = C.POINTER(C.c_float)

# (name, restype, argtypes) for every symbol declared in include/nexel_b200.h
SIGNATURES = [
    ("nx_version", C.c_char_p, []),
    ("nx_status_name", C.c_char_p, [C.c_int]),
    ("nx_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("nx_ctx_create", C.c_int, [C.c_int, C.POINTER(P)]),
    ("nx_ctx_destroy", None, [P]),
    ("nx_ctx_last_error", C.c_char_p, [P, C.POINTER(C.c_int)]),
    ("nx_ctx_stream", P, [P]),
    ("nx_ctx_synchronize", C.c_int, [P]),
    ("nx_ctx_join", C.c_int, [P]),
    ("nx_ctx_set_profiling", C.c_int, [P, C.c_int]),
    ("nx_ctx_stage_times", C.c_int, [P, PF, C.c_int, C.POINTER(C.c_int)]),
    ("nx_stage_name", C.c_char_p, [C.c_int]),
    ("nx_launch_count", C.c_uint64, []),
    ("nx_scene_create", C.c_int,
     [P, C.POINTER(nx_settings), I64, PD, C.POINTER(nx_field_desc), PD, PD, PD, PD, C.POINTER(P)]),
    ("nx_scene_set_settings", C.c_int, [P, P, C.POINTER(nx_settings)]),
    ("nx_scene_load_nexl", C.c_int, [P, C.c_char_p, C.POINTER(P), C.POINTER(nx_nexl_info)]),
    ("nx_nexl_cameras", C.c_int, [C.c_char_p, C.POINTER(nx_camera), C.c_void_p, C.c_int, C.POINTER(C.c_int)]),
    ("nx_scene_get_settings", C.c_int, [P, C.POINTER(nx_settings)]),
    ("nx_scene_destroy", None, [P]),
    ("nx_frame_create", C.c_int, [P, C.c_int, C.c_int, C.c_int, C.POINTER(P)]),
    ("nx_frame_destroy", None, [P]),
    ("nx_frame_view_get", C.c_int, [P, C.POINTER(nx_frame_view)]),
    ("nx_frame_download", C.c_int, [P, P, C.POINTER(nx_host_frame), P]),
    ("nx_frame_upload", C.c_int, [P, P, C.c_int, C.c_int, C.c_int, C.POINTER(nx_host_frame), P]),
    ("nx_frame_stats_get", C.c_int, [P, P, C.POINTER(nx_frame_stats)]),
    ("nx_collection_pass", C.c_int, [P, P, C.POINTER(nx_camera), P, P]),
    ("nx_texturing_pass", C.c_int, [P, P, C.POINTER(nx_camera), P, P]),
    ("nx_render_views", C.c_int, [P, P, C.POINTER(nx_camera), C.c_int, C.POINTER(P), C.c_int, P]),
    ("nx_render", C.c_int, [P, P, C.POINTER(nx_camera), P, P]),
    ("nx_frame_set_backward", C.c_int, [P, P, C.c_int]),
    ("nx_render_backward", C.c_int,
     [P, P, C.POINTER(nx_camera), P, C.POINTER(nx_upstream), C.POINTER(nx_grads), P, P, P]),
    ("nx_render_backward_host", C.c_int,
     [P, P, C.POINTER(nx_camera), P, C.POINTER(nx_upstream), C.POINTER(nx_grads), PD, PD]),
    ("nx_loss_weights_default", None, [C.POINTER(nx_loss_weights)]),
    ("nx_losses_backward", C.c_int,
     [P, P, P, P, C.POINTER(nx_loss_weights), P, P, P, C.POINTER(nx_grads), P, P]),
    ("nx_losses_backward_opt", C.c_int,
     [P, P, P, P, C.POINTER(nx_loss_weights), P, P, P, C.POINTER(nx_grads), P, P, P]),
    ("nx_losses_backward_host", C.c_int,
     [P, P, P, PD, C.POINTER(nx_loss_weights), PD, PD, PD, C.POINTER(nx_grads), C.POINTER(nx_loss_terms)]),
    ("nx_optimizer_create", C.c_int, [P, P, C.POINTER(P)]),
    ("nx_optimizer_destroy", None, [P]),
    ("nx_optimizer_step", C.c_int, [P, P, P, C.POINTER(nx_grads), C.POINTER(nx_adam_config), P]),
    ("nx_optimizer_steps", C.c_int, [P, PI64]),
    ("nx_optimizer_size", C.c_int, [P, C.c_int, PI64]),
    ("nx_optimizer_set_params", C.c_int, [P, P, P, C.c_int, PD, I64]),
    ("nx_optimizer_download", C.c_int, [P, P, P, C.c_int, PD, PD, PD]),
    ("nx_pixel_error", C.c_int, [P, P, P, P, P]),
    ("nx_scene_download", C.c_int, [P, P, PD, PD, PD, PD, PD]),
    ("nx_scene_prune", C.c_int, [P, P, P, D, P, PI64]),
    ("nx_scene_densify_split", C.c_int, [P, P, P, P, P, I64, D, P, PI64, PI64]),
    ("nx_debug_tile_lists", C.c_int,
     [P, P, C.POINTER(nx_camera), C.c_int, PI64, PI32, I64, PI64, PI32, PI32]),
    ("nx_debug_pixel_hits", C.c_int, [P, P, C.POINTER(nx_camera), C.c_int, C.c_int, C.c_int, PI32, PI32]),
    ("nx_debug_fastmath", C.c_int, [C.c_int, PD, PD, I64]),
    ("nx_debug_radix_sort", C.c_int, [C.c_int, P, PI32, I64, I64, C.c_int, C.c_int]),
    ("nx_debug_scan", C.c_int, [PI32, PI32, I64, I64, PI32]),
    ("nx_synth_stump_like", C.c_int,
     [I64, D, C.c_uint64, D, I32, D, C.c_uint64, PD, C.POINTER(nx_settings), C.POINTER(nx_field_desc), PD, PD,
      PD, PD]),
    ("nx_synth_ring_camera", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(nx_camera)]),
    ("nx_settings_default", None, [C.POINTER(nx_settings)]),
]

_lib = None


def load(path: str | None = None):
    """Load libnexel_b200.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(
            f"{p} not found: the sm_100a render library is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'` or `make lib`)")
    lib = C.CDLL(p)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
