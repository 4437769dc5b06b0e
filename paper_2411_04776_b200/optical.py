"""Batched mirrors of the reference optical functions (REF/optical.py).

``shade`` here is kernel (b): it shades a smoothed indentation map through the
binned 125x180 LUT of the north star.  The reference's global
polynomial ``PolyTable`` is the single-bin special case (``lut_from_polytable``).
"""

import numpy as np
import torch

from . import _lib
from .config import PipelineConfig
from .context import blur_config, context_for, require
from .tactile import HeightMap, IndentationMap


def normals_from(source, pixel_pitch=None) -> torch.Tensor:
    """Unit normals [N, H, W, 3] from np.gradient-style differences
    (REF/optical.py:138-163).  A HeightMap is negated, an IndentationMap used
    as is, a raw tensor needs ``pixel_pitch``."""
    from .errors import InvalidArgumentError

    if isinstance(source, HeightMap):
        elev, pitch = -source.values, source.pixel_pitch
    elif isinstance(source, IndentationMap):
        elev, pitch = source.values, source.pixel_pitch
    else:
        if pixel_pitch is None:
            raise InvalidArgumentError("pixel_pitch required for raw arrays")
        elev, pitch = source, pixel_pitch
    if elev.dim() not in (2, 3):
        raise InvalidArgumentError("elevation field must be 2-D")
    single = elev.dim() == 2
    v = (elev.unsqueeze(0) if single else elev).contiguous().float()
    n, h, w = v.shape
    if h < 2 or w < 2:
        raise InvalidArgumentError("gradient needs at least 2 samples per axis")
    ctx = context_for(blur_config(h, w, pitch, 1.0, ((0.0, 0),)), v.device)
    out = torch.empty((n, h, w, 3), dtype=torch.float32, device=v.device)
    _lib.check(ctx.lib.tac_normals(ctx.handle, v.data_ptr(), out.data_ptr(), n, ctx.stream()),
               "tac_normals")
    return out[0] if single else out


def shade(smoothed, cfg: PipelineConfig) -> torch.Tensor:
    """Kernel (b): smoothed indentation [N, H, W] -> uint8 RGB [N, H, W, 3].

    gradient (REF/optical.py:160) -> bins -> per-bin quadratic in (nx, ny)
    (basis REF/optical.py:82-88, c0 cancels as REF/optical.py:244) -> + bg ->
    rint -> clamp (uint8 rule REF/cli.py:134-139)."""
    v = smoothed.values if isinstance(smoothed, IndentationMap) else smoothed
    single = v.dim() == 2
    v = (v.unsqueeze(0) if single else v).contiguous()
    ctx = context_for(cfg, v.device)
    n = v.shape[0]
    require(v, "smoothed", torch.float32, (n, ctx.H, ctx.W), ctx.device)
    out = torch.empty((n, ctx.H, ctx.W, 3), dtype=torch.uint8, device=v.device)
    _lib.check(ctx.lib.tac_shade(ctx.handle, v.data_ptr(), out.data_ptr(), n, ctx.stream()), "tac_shade")
    return out[0] if single else out


def lut_from_polytable(coeffs, mag_bins=125, dir_bins=180, scale=255.0) -> np.ndarray:
    """Degenerate binned LUT: every bin holds the reference global table
    (PolyTable.coeffs, REF/optical.py:97-135) in 8-bit units."""
    c = np.asarray(coeffs, dtype=np.float64)
    if c.shape != (3, 6):
        from .errors import InvalidArgumentError

        raise InvalidArgumentError("coeffs must be (3, 6) for degree 2")
    return np.broadcast_to((c * scale).astype(np.float32), (mag_bins, dir_bins, 3, 6)).copy()
