"""Batched mirrors of the reference tactile-map functions (REF/tactile.py).

Maps are torch CUDA tensors with a leading env dimension ([N, H, W]); a
single [H, W] map is accepted and returned unbatched.  Every computation is a
``libtac_b200.so`` call; nothing here computes on the CPU.
"""

from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _lib
from .config import DEFAULT_PYRAMID, levels_from_kernel_sizes, levels_from_sigmas
from .context import blur_config, context_for, require
from .errors import InvalidArgumentError


@dataclass
class HeightMap:
    """Per-pixel depth from the camera plane, metres (REF/tactile.py:72-87).

    ``validate=True`` runs the reference's eager checks (2-D per env, finite,
    positive pitch); the finiteness check synchronises the device.
    """

    values: torch.Tensor
    pixel_pitch: float
    validate: bool = True

    def __post_init__(self):
        _check_map(self.values, self.pixel_pitch, self.validate, "height map", nonneg=False)


@dataclass
class IndentationMap:
    """Per-pixel penetration, metres, >= 0 (REF/tactile.py:90-107)."""

    values: torch.Tensor
    pixel_pitch: float
    validate: bool = True

    def __post_init__(self):
        _check_map(self.values, self.pixel_pitch, self.validate, "indentation", nonneg=True)


def _check_map(v, pitch, validate, what, nonneg):
    if not isinstance(v, torch.Tensor):
        raise InvalidArgumentError(f"{what} values must be a torch.Tensor")
    if v.dim() not in (2, 3):
        raise InvalidArgumentError(f"{what} values must be 2-D (or [N, H, W])")
    if not pitch > 0:
        raise InvalidArgumentError("pixel_pitch must be positive")
    if validate and v.numel():
        if not bool(torch.isfinite(v).all()):
            raise InvalidArgumentError(f"{what} values must be finite")
        if nonneg and bool((v < 0).any()):
            raise InvalidArgumentError(f"{what} values must be >= 0")


def _batched(v):
    v = v.contiguous()
    if v.dtype != torch.float32:
        v = v.float()
    return (v.unsqueeze(0), True) if v.dim() == 2 else (v, False)


def indentation_from(hm: HeightMap, cfg) -> IndentationMap:
    """ind = clip(rest - depth, 0, rest), REF/tactile.py:193-197."""
    v, single = _batched(hm.values)
    n, h, w = v.shape
    ctx = context_for(blur_config(h, w, hm.pixel_pitch, cfg.gelpad_thickness, ((0.0, 0),)), v.device)
    out = torch.empty_like(v)
    _lib.check(ctx.lib.tac_indentation(ctx.handle, v.data_ptr(), out.data_ptr(), n, ctx.stream()),
               "tac_indentation")
    return IndentationMap(out[0] if single else out, hm.pixel_pitch, validate=False)


def smooth_pyramid(
    ind: IndentationMap,
    kernel_sizes: Sequence[int] = DEFAULT_PYRAMID,
    sigmas: Optional[Sequence[float]] = None,
) -> IndentationMap:
    """Mean of replicate-padded Gaussian blurs, REF/tactile.py:200-222.

    ``kernel_sizes`` follows the reference parameterisation (odd k,
    sigma = k/6, radius (k-1)//2); ``sigmas`` selects the north star's
    sigma-keyed pyramid (radius ceil(3 sigma)).
    """
    levels = levels_from_sigmas(sigmas) if sigmas is not None else levels_from_kernel_sizes(kernel_sizes)
    v, single = _batched(ind.values)
    n, h, w = v.shape
    ctx = context_for(blur_config(h, w, ind.pixel_pitch, 1.0, levels), v.device)
    out = torch.empty_like(v)
    _lib.check(
        ctx.lib.tac_contact_blur(ctx.handle, v.data_ptr(), _lib.TAC_INPUT_INDENTATION, out.data_ptr(),
                                 None, None, n, ctx.stream()),
        "tac_contact_blur",
    )
    return IndentationMap(out[0] if single else out, ind.pixel_pitch, validate=False)


def contact_blur(depth: torch.Tensor, cfg, *, input_kind="depth", summary=True):
    """Kernel (a) on its own: clamp + pyramid (+ contact summary) for a
    PipelineConfig ``cfg``.  Returns (blurred [N,H,W], summary [N,8] or None)."""
    ctx = context_for(cfg, depth.device)
    n = depth.shape[0]
    require(depth, "depth", torch.float32, (n, ctx.H, ctx.W), ctx.device)
    out = torch.empty_like(depth)
    summ = torch.empty((n, 8), dtype=torch.float32, device=depth.device) if summary else None
    ws = ctx.workspace(n) if summary else None
    kind = _lib.TAC_INPUT_DEPTH if input_kind == "depth" else _lib.TAC_INPUT_INDENTATION
    _lib.check(
        ctx.lib.tac_contact_blur(ctx.handle, depth.data_ptr(), kind, out.data_ptr(),
                                 summ.data_ptr() if summary else None,
                                 ws.data_ptr() if summary else None, n, ctx.stream()),
        "tac_contact_blur",
    )
    return out, summ


def _camera_frame(points, sensor_pose):
    """World -> camera frame like the reference (REF/tactile.py:141-146): the
    inverse sensor pose applied as p @ R^T + t in float64.  ``sensor_pose``:
    None (identity), an object with ``inverse().apply`` (e.g. a tacsim Pose),
    or a 4x4 camera-to-world matrix."""
    import numpy as np

    p = np.asarray(points, dtype=np.float64)
    if sensor_pose is None:
        return p
    if hasattr(sensor_pose, "inverse"):
        return np.asarray(sensor_pose.inverse().apply(p), dtype=np.float64)
    m = np.asarray(sensor_pose, dtype=np.float64)
    if m.shape != (4, 4):
        raise InvalidArgumentError("sensor_pose must be None, a Pose, or a 4x4 matrix")
    rinv = m[:3, :3].T
    return p @ rinv.T + (-(rinv @ m[:3, 3]))


def render_heightmap(surfaces, sensor_pose, cfg) -> HeightMap:
    """Orthographic z-buffer render, REF/tactile.py:129-190, on the GPU.

    Mirrors the reference call for one sensor: ``surfaces`` is a sequence of
    (vertices [V,3] world frame, triangles [T,3]) pairs; ``sensor_pose`` as in
    ``_camera_frame``; ``cfg`` a SensorConfig or PipelineConfig.  Returns a
    HeightMap [H, W] (fp32 on the GPU) equal to fp32 of the reference's
    float64 depth.  Batched use: ``render_heightmaps``.
    """
    import numpy as np

    sensor = getattr(cfg, "sensor", cfg)
    verts, tris, base = [], [], 0
    for item in surfaces:
        if not (isinstance(item, (tuple, list)) and len(item) == 2):
            raise InvalidArgumentError("surface must be (vertices, triangles)")
        v = np.asarray(item[0], dtype=np.float64)
        t = np.asarray(item[1], dtype=np.int64)
        if v.ndim != 2 or v.shape[1] != 3:
            raise InvalidArgumentError("surface vertices must be (n, 3)")
        if t.ndim != 2 or t.shape[1] != 3:
            raise InvalidArgumentError("surface triangles must be (m, 3)")
        verts.append(_camera_frame(v, sensor_pose))
        tris.append(t + base)
        base += len(v)
    v = np.concatenate(verts) if verts else np.zeros((0, 3))
    t = np.concatenate(tris) if tris else np.zeros((0, 3), np.int64)
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
    out = render_heightmaps(torch.as_tensor(v, device=dev)[None], torch.as_tensor(t, device=dev), sensor)
    return HeightMap(out[0], sensor.pixel_pitch, validate=False)


def render_heightmaps(verts: torch.Tensor, tris: torch.Tensor, sensor, out: Optional[torch.Tensor] = None):
    """Batched z-buffer (kernel ``raster_kernel``): ``verts`` fp64 [N, V, 3]
    camera-frame vertices (one set per env, e.g. one mesh at N poses),
    ``tris`` [T, 3] shared triangle indices.  Returns depth fp32 [N, H, W]."""
    sensor = getattr(sensor, "sensor", sensor)
    h, w = sensor.image_size
    if verts.dim() != 3 or verts.shape[-1] != 3:
        raise InvalidArgumentError("verts must be [N, V, 3]")
    if tris.dim() != 2 or tris.shape[-1] != 3:
        raise InvalidArgumentError("tris must be [T, 3]")
    n, nv = verts.shape[0], verts.shape[1]
    if tris.numel() and (int(tris.min()) < 0 or int(tris.max()) >= nv):
        raise InvalidArgumentError("triangle index out of range")
    v = verts.to(torch.float64).contiguous()
    t = tris.to(device=v.device, dtype=torch.int32).contiguous()
    ctx = context_for(blur_config(h, w, sensor.pixel_pitch, sensor.gelpad_thickness, ((0.0, 0),)), v.device)
    if out is None:
        out = torch.empty((n, h, w), dtype=torch.float32, device=v.device)
    require(out, "out", torch.float32, (n, h, w), ctx.device)
    _lib.check(ctx.lib.tac_render_heightmap(ctx.handle, v.data_ptr(), nv, t.data_ptr(), t.shape[0],
                                            out.data_ptr(), n, ctx.stream()), "tac_render_heightmap")
    return out
