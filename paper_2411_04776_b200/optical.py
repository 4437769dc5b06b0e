"""Batched mirrors of the reference optical functions (REF/optical.py).

``shade`` here is kernel (b): it shades a smoothed indentation map through the
binned 125x180 LUT of the north star.  The reference's global
polynomial ``PolyTable`` is the single-bin special case (``lut_from_polytable``).
"""

import logging

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


log = logging.getLogger(__name__)
_SATURATION_WARN_FRACTION = 0.01  # REF/optical.py:29


def shade(smoothed, cfg: PipelineConfig, *, warn_saturation: bool = True) -> torch.Tensor:
    """Kernel (b): smoothed indentation [N, H, W] -> uint8 RGB [N, H, W, 3].

    gradient (REF/optical.py:160) -> bins -> per-bin quadratic in (nx, ny)
    (basis REF/optical.py:82-88, c0 cancels as REF/optical.py:244) -> + bg ->
    rint -> clamp (uint8 rule REF/cli.py:134-139).  Like the reference, logs a
    warning for a frame whose clip changed more than 1 % of the channel values
    (REF/optical.py:246-249); that check reads a per-env count back from the
    device (``warn_saturation=False`` skips it)."""
    v = smoothed.values if isinstance(smoothed, IndentationMap) else smoothed
    single = v.dim() == 2
    v = (v.unsqueeze(0) if single else v).contiguous()
    ctx = context_for(cfg, v.device)
    n = v.shape[0]
    require(v, "smoothed", torch.float32, (n, ctx.H, ctx.W), ctx.device)
    out = torch.empty((n, ctx.H, ctx.W, 3), dtype=torch.uint8, device=v.device)
    sat = torch.empty((n,), dtype=torch.int32, device=v.device) if warn_saturation and n else None
    _lib.check(ctx.lib.tac_shade_ex(ctx.handle, v.data_ptr(), out.data_ptr(),
                                    sat.data_ptr() if sat is not None else None, n, ctx.stream()), "tac_shade")
    if sat is not None:
        frac = sat.double().cpu() / (3.0 * ctx.H * ctx.W)
        for i in torch.nonzero(frac > _SATURATION_WARN_FRACTION).flatten().tolist():
            log.warning("shade: %.1f%% of pixels saturated (env %d)", 100.0 * float(frac[i]), i)
    return out[0] if single else out


def lut_from_polytable(coeffs, mag_bins=125, dir_bins=180, scale=255.0) -> np.ndarray:
    """Degenerate binned LUT: every bin holds the reference global table
    (PolyTable.coeffs, REF/optical.py:97-135) in 8-bit units."""
    c = np.asarray(coeffs, dtype=np.float64)
    if c.shape != (3, 6):
        from .errors import InvalidArgumentError

        raise InvalidArgumentError("coeffs must be (3, 6) for degree 2")
    return np.broadcast_to((c * scale).astype(np.float32), (mag_bins, dir_bins, 3, 6)).copy()


_SHADOW_CFGS = {}


def _shadow_config(h, w, pitch, directions, factor, max_steps, softness):
    from .config import SensorConfig

    dirs = np.asarray(directions, dtype=np.float64)
    key = (h, w, float(pitch), dirs.tobytes(), float(factor), int(max_steps), float(softness))
    cfg = _SHADOW_CFGS.get(key)
    if cfg is None:
        cfg = PipelineConfig(
            sensor=SensorConfig.from_pitch(h, w, pitch), levels=((0.0, 0),),
            lut=np.zeros((1, 1, 3, 6), np.float32), background=np.zeros((h, w, 3), np.float32),
            light_dirs=dirs, shadow_factor=factor, shadow_steps=max_steps, shadow_softness=softness,
        )
        _SHADOW_CFGS[key] = cfg
    return cfg


def shadow_factor(hm: HeightMap, directions, factor=0.6, max_steps=80, softness=5e-5) -> torch.Tensor:
    """Multiplicative shadow factor [N, H, W] of add_shadows (REF/optical.py:261-300)
    for the light directions (n, 3) (e.g. a LightingModel's ``directions``)."""
    from .errors import InvalidArgumentError

    if not 0.0 <= factor <= 1.0:
        raise InvalidArgumentError("shadow factor must be in [0, 1]")
    v = hm.values
    single = v.dim() == 2
    v = (v.unsqueeze(0) if single else v).contiguous().float()
    n, h, w = v.shape
    cfg = _shadow_config(h, w, hm.pixel_pitch, directions, factor, max_steps, softness)
    ctx = context_for(cfg, v.device)
    out = torch.empty((n, h, w), dtype=torch.float32, device=v.device)
    if not cfg.shadows:
        out.fill_(1.0)
    else:
        _lib.check(ctx.lib.tac_shadow(ctx.handle, v.data_ptr(), _lib.TAC_INPUT_DEPTH, out.data_ptr(), None, n,
                                      ctx.stream()), "tac_shadow")
    return out[0] if single else out


def add_shadows(rgb, hm: HeightMap, directions, factor=0.6, max_steps=80, softness=5e-5) -> torch.Tensor:
    """Mirror of add_shadows (REF/optical.py:261-300): returns a darkened copy of
    the float RGB [N, H, W, 3] (or [H, W, 3]); factor 1.0 is the identity."""
    from .errors import InvalidArgumentError

    if not 0.0 <= factor <= 1.0:
        raise InvalidArgumentError("shadow factor must be in [0, 1]")
    img = rgb.detach().clone().float().contiguous()
    single = img.dim() == 3
    if single:
        img = img.unsqueeze(0)
    v = hm.values
    v = (v.unsqueeze(0) if v.dim() == 2 else v).contiguous().float()
    if tuple(img.shape[:3]) != tuple(v.shape):
        raise InvalidArgumentError("image and height map shapes differ")
    n, h, w = v.shape
    cfg = _shadow_config(h, w, hm.pixel_pitch, directions, factor, max_steps, softness)
    if cfg.shadows:
        ctx = context_for(cfg, v.device)
        _lib.check(ctx.lib.tac_shadow(ctx.handle, v.data_ptr(), _lib.TAC_INPUT_DEPTH, None, img.data_ptr(), n,
                                      ctx.stream()), "tac_shadow")
    return img[0] if single else img
