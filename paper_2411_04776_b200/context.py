"""Owning wrapper of a ``tac_ctx`` plus per-stream workspaces.

PyTorch is plumbing here: it allocates device buffers and supplies the CUDA
stream; every computation is a call into ``libtac_b200.so``.
"""

import ctypes
import threading
import weakref

import numpy as np
import torch

from . import _lib
from .config import PipelineConfig
from .errors import InvalidArgumentError


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream_handle(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def require(t, name, dtype, shape, device):
    """Shape/dtype/device/contiguity checks -> InvalidArgumentError."""
    if not isinstance(t, torch.Tensor):
        raise InvalidArgumentError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise InvalidArgumentError(f"{name} must be {dtype}, got {t.dtype}")
    if t.device != device:
        raise InvalidArgumentError(f"{name} must be on {device}, got {t.device}")
    if tuple(t.shape) != tuple(shape):
        raise InvalidArgumentError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise InvalidArgumentError(f"{name} must be contiguous")
    return t


class Context:
    """One uploaded ``PipelineConfig`` on one CUDA device."""

    def __init__(self, cfg: PipelineConfig, device=None):
        if not torch.cuda.is_available():
            raise _lib.NativeLibraryError("CUDA device required: the tactile path has no CPU fallback")
        self.lib = _lib.load()
        self.cfg = cfg
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.type != "cuda":
            raise InvalidArgumentError(f"device must be a CUDA device, got {dev}")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        s = cfg.sensor
        c = _lib.TacConfig()
        c.height, c.width = int(s.image_size[0]), int(s.image_size[1])
        c.pixel_pitch = float(s.pixel_pitch)
        c.gel_thickness = float(s.gelpad_thickness)
        if len(cfg.levels) > _lib.TAC_MAX_LEVELS:
            raise _lib.UnsupportedConfigError(f"at most {_lib.TAC_MAX_LEVELS} pyramid levels")
        c.n_levels = len(cfg.levels)
        for i, (sig, rad) in enumerate(cfg.levels):
            c.sigma[i] = float(sig)
            c.radius[i] = int(rad)
        c.mag_bins, c.dir_bins = int(cfg.lut.shape[0]), int(cfg.lut.shape[1])
        c.g_max = float(cfg.g_max)
        self._lut = cfg.lut  # keep host arrays alive during create
        self._bg = cfg.background
        self._grid = cfg.rest_grid
        c.lut = self._lut.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        c.background = self._bg.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        c.rest_grid = self._grid.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        c.marker_rows, c.marker_cols = int(s.marker_grid[0]), int(s.marker_grid[1])
        mp = cfg.marker_params
        c.k_n, c.lambda_n, c.lambda_s, c.k_t, c.lambda_t = (
            mp.k_n, mp.lambda_n, mp.lambda_s, mp.k_t, mp.lambda_t)
        c.contact_threshold = float(cfg.contact_threshold)
        c.dot_radius = int(cfg.dot_radius)
        for i in range(3):
            c.dot_color[i] = int(cfg.dot_color[i])
        c.n_lights = len(cfg.light_dirs)
        for l, d in enumerate(cfg.light_dirs):
            for q in range(3):
                c.light_dir[l][q] = float(d[q])
        c.shadow_factor = float(cfg.shadow_factor)
        c.shadow_steps = int(cfg.shadow_steps)
        c.shadow_softness = float(cfg.shadow_softness)
        c.lut_dtype = {"f32": _lib.TAC_LUT_F32, "f16": _lib.TAC_LUT_F16}[cfg.lut_dtype]
        c.kernel_path = {"auto": _lib.TAC_PATH_AUTO, "band": _lib.TAC_PATH_BAND,
                         "fused": _lib.TAC_PATH_FUSED, "stream": _lib.TAC_PATH_STREAM}[cfg.kernel_path]
        c.chunk_envs = int(cfg.chunk_envs)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.tac_ctx_create(ctypes.byref(c), ctypes.byref(handle)), "tac_ctx_create")
        self.handle = handle
        self._finalizer = weakref.finalize(self, self.lib.tac_ctx_destroy, handle)
        self._ws = {}
        self._ws_lock = threading.Lock()
        self.H, self.W = c.height, c.width
        self.rows, self.cols = c.marker_rows, c.marker_cols

    # -- workspaces ---------------------------------------------------------
    def workspace(self, n_env):
        """Workspace for the current stream (the library initialises what it
        uses on every call).  Calls from several host threads on ONE stream
        share it and must not overlap: use one stream per thread."""
        stream = torch.cuda.current_stream(self.device)
        key = stream.cuda_stream
        nbytes = int(self.lib.tac_workspace_bytes(self.handle, int(n_env)))
        with self._ws_lock:
            ws = self._ws.get(key)
            if ws is None or ws.numel() < nbytes:
                ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
                self._ws[key] = ws
        return ws

    @property
    def tiles_per_frame(self):
        return int(self.lib.tac_tiles_per_frame(self.handle))

    def stream(self):
        return _stream_handle(self.device)

    def close(self):
        self._finalizer()


_CACHE = {}
_CACHE_LOCK = threading.Lock()


def context_for(cfg: PipelineConfig, device=None) -> Context:
    """Contexts are cached per (config object, device)."""
    if not torch.cuda.is_available():
        raise _lib.NativeLibraryError("CUDA device required: the tactile path has no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (id(cfg), dev.index)
    with _CACHE_LOCK:
        hit = _CACHE.get(key)
        if hit is not None and hit[0]() is cfg:
            return hit[1]
        ctx = Context(cfg, dev)
        _CACHE[key] = (weakref.ref(cfg), ctx)
        return ctx


def blur_config(h, w, pitch, rest, levels):
    """Minimal PipelineConfig for the pyramid-only mirrors (dummy 1x1 LUT)."""
    from .config import SensorConfig

    key = ("blur", h, w, float(pitch), float(rest), tuple(levels))
    with _CACHE_LOCK:
        cfg = _BLUR_CFGS.get(key)
        if cfg is None:
            cfg = PipelineConfig(
                sensor=SensorConfig.from_pitch(h, w, pitch, rest),
                levels=tuple(levels),
                lut=np.zeros((1, 1, 3, 6), np.float32),
                background=np.zeros((h, w, 3), np.float32),
            )
            _BLUR_CFGS[key] = cfg
    return cfg


_BLUR_CFGS = {}
