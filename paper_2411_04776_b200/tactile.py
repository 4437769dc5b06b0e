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
