"""ctypes binding of ``libtac_b200.so`` (the C ABI in ``include/tac_b200.h``).

The library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_2411_04776_b200/csrc``.  Loading fails loudly when it is
missing: there is no CPU fallback on the product path.
"""

import ctypes
import os
import threading

from .errors import InvalidArgumentError, NativeLibraryError, UnsupportedConfigError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TAC_B200_LIB", os.path.join(_HERE, "libtac_b200.so"))

TAC_OK = 0
TAC_ERR_INVALID = 1
TAC_ERR_CUDA = 2
TAC_ERR_UNSUPPORTED = 3
TAC_MAX_LEVELS = 8
TAC_MAX_RADIUS = 24
TAC_MAX_LIGHTS = 4
TAC_MAX_SHADOW_STEPS = 256
TAC_INPUT_DEPTH = 0
TAC_INPUT_INDENTATION = 1
TAC_LOAD_GIVEN = 0
TAC_LOAD_TRACK = 1
TAC_LUT_F32 = 0
TAC_LUT_F16 = 1
TAC_PATH_AUTO = 0
TAC_PATH_BAND = 1
TAC_PATH_FUSED = 2
TAC_PATH_STREAM = 3
TAC_TIMING_KINDS = 4

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64


class TacConfig(ctypes.Structure):
    """struct tac_config (include/tac_b200.h); struct_size is filled in."""

    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("height", _i32),
        ("width", _i32),
        ("pixel_pitch", ctypes.c_double),
        ("gel_thickness", ctypes.c_double),
        ("n_levels", _i32),
        ("sigma", ctypes.c_double * TAC_MAX_LEVELS),
        ("radius", _i32 * TAC_MAX_LEVELS),
        ("mag_bins", _i32),
        ("dir_bins", _i32),
        ("g_max", ctypes.c_double),
        ("lut", ctypes.POINTER(ctypes.c_float)),
        ("background", ctypes.POINTER(ctypes.c_float)),
        ("marker_rows", _i32),
        ("marker_cols", _i32),
        ("rest_grid", ctypes.POINTER(ctypes.c_double)),
        ("k_n", ctypes.c_double),
        ("lambda_n", ctypes.c_double),
        ("lambda_s", ctypes.c_double),
        ("k_t", ctypes.c_double),
        ("lambda_t", ctypes.c_double),
        ("contact_threshold", ctypes.c_double),
        ("dot_radius", _i32),
        ("dot_color", ctypes.c_uint8 * 3),
        ("n_lights", _i32),
        ("light_dir", (ctypes.c_double * 3) * TAC_MAX_LIGHTS),
        ("shadow_factor", ctypes.c_double),
        ("shadow_steps", _i32),
        ("shadow_softness", ctypes.c_double),
        ("lut_dtype", _i32),
        ("kernel_path", _i32),
        ("chunk_envs", _i32),
    ]

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.struct_size = ctypes.sizeof(TacConfig)


class TacPipelineArgs(ctypes.Structure):
    """struct tac_pipeline_args (include/tac_b200.h); struct_size is filled in."""

    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("in_", _p),
        ("input_kind", _i32),
        ("load_mode", _i32),
        ("shear", _p),
        ("twist", _p),
        ("state", _p),
        ("pose_delta", _p),
        ("rgb", _p),
        ("disp", _p),
        ("summary", _p),
        ("contact", _p),
        ("blurred", _p),
        ("shadow", _p),
        ("splat", _i32),
        ("saturated", _p),
        ("workspace", _p),
        ("n_env", _i64),
    ]

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.struct_size = ctypes.sizeof(TacPipelineArgs)


# name -> (restype, argtypes); every symbol include/tac_b200.h declares.
SIGNATURES = {
    "tac_ctx_create": (ctypes.c_int, [ctypes.POINTER(TacConfig), ctypes.POINTER(_p)]),
    "tac_ctx_destroy": (ctypes.c_int, [_p]),
    "tac_last_error": (ctypes.c_char_p, []),
    "tac_workspace_bytes": (ctypes.c_size_t, [_p, _i64]),
    "tac_tiles_per_frame": (_i32, [_p]),
    "tac_pipeline_path": (_i32, [_p]),
    "tac_pipeline_launches": (_i32, [_p, _i64]),
    "tac_pipeline_profile": (ctypes.c_int, [_p, ctypes.POINTER(TacPipelineArgs), _p, _i32, _p]),
    "tac_timing_begin": (ctypes.c_int, [_p, _i32]),
    "tac_timing_end": (ctypes.c_int, [_p, _p, _p]),
    "tac_render_heightmap": (ctypes.c_int, [_p, _p, _i64, _p, _i64, _p, _i64, _p]),
    "tac_indentation": (ctypes.c_int, [_p, _p, _p, _i64, _p]),
    "tac_contact_blur": (ctypes.c_int, [_p, _p, _i32, _p, _p, _p, _i64, _p]),
    "tac_normals": (ctypes.c_int, [_p, _p, _p, _i64, _p]),
    "tac_shade": (ctypes.c_int, [_p, _p, _p, _i64, _p]),
    "tac_shade_ex": (ctypes.c_int, [_p, _p, _p, _p, _i64, _p]),
    "tac_contact": (ctypes.c_int, [_p, _p, _i32, _p, _p, _p, _i64, _p]),
    "tac_track_load": (ctypes.c_int, [_p, _p, _p, _p, _i64, _p]),
    "tac_marker_displacements": (ctypes.c_int, [_p, _p, _p, _i64, _p]),
    "tac_render_markers": (ctypes.c_int, [_p, _p, _p, _i64, _p]),
    "tac_shadow": (ctypes.c_int, [_p, _p, _i32, _p, _p, _i64, _p]),
    "tac_pipeline": (ctypes.c_int, [_p, ctypes.POINTER(TacPipelineArgs), _p]),
}

_lib = None
_lock = threading.Lock()


def load(path=None):
    """Load (once) and return the ctypes handle; raises NativeLibraryError."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise NativeLibraryError(
                f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_2411_04776_b200/csrc` (no CPU fallback exists)"
            )
        try:
            lib = ctypes.CDLL(p)
        except OSError as e:  # pragma: no cover - depends on the box
            raise NativeLibraryError(f"cannot load {p}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def last_error():
    msg = load().tac_last_error()
    return msg.decode() if msg else ""


def check(status, what=""):
    """Map a C ABI status onto the reference error classes."""
    if status == TAC_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == TAC_ERR_INVALID:
        raise InvalidArgumentError(msg)
    if status == TAC_ERR_UNSUPPORTED:
        raise UnsupportedConfigError(msg)
    raise NativeLibraryError(msg)
