"""Batched mirrors of the reference marker functions (REF/marker.py).

Loads use the fp64 LoadState layout of include/tac_b200.h:
[N, 8] = (c_x, c_y, d_c, s_x, s_y, twist, in_contact, 0).
Marker geometry, model constants, threshold and dot style come from a
``PipelineConfig`` (``marker_config`` builds a minimal one).
"""

import numpy as np
import torch

from . import _lib
from .config import DEFAULT_CONTACT_THRESHOLD, MarkerParams, PipelineConfig, SensorConfig
from .context import context_for, require
from .errors import InvalidArgumentError
from .tactile import IndentationMap

LOAD_FIELDS = ("cx", "cy", "dmax", "sx", "sy", "twist", "in_contact", "pad")

_MCFG = {}


def marker_config(sensor: SensorConfig, params: MarkerParams = MarkerParams(),
                  threshold: float = DEFAULT_CONTACT_THRESHOLD, dot_radius: int = 4,
                  dot_color=(25, 25, 25), rest_grid=None) -> PipelineConfig:
    """Minimal PipelineConfig for the marker-only mirrors (cached by value)."""
    key = (sensor, params, float(threshold), int(dot_radius), tuple(dot_color),
           None if rest_grid is None else np.asarray(rest_grid, np.float64).tobytes())
    cfg = _MCFG.get(key)
    if cfg is None:
        h, w = sensor.image_size
        cfg = PipelineConfig(
            sensor=sensor, levels=((0.0, 0),), lut=np.zeros((1, 1, 3, 6), np.float32),
            background=np.zeros((h, w, 3), np.float32), marker_params=params,
            contact_threshold=threshold, dot_radius=dot_radius, dot_color=tuple(dot_color),
            rest_grid=rest_grid,
        )
        _MCFG[key] = cfg
    return cfg


def contact_center(ind, cfg: PipelineConfig, *, input_kind="indentation"):
    """Indentation-weighted centroid over ind > threshold, REF/marker.py:103-121.

    Returns (contact [N, 8] fp64 LoadState with zero shear/twist,
    summary [N, 8] fp32)."""
    if threshold_invalid(cfg.contact_threshold):
        raise InvalidArgumentError("threshold must be positive")
    v = ind.values if isinstance(ind, IndentationMap) else ind
    single = v.dim() == 2
    v = (v.unsqueeze(0) if single else v).contiguous()
    ctx = context_for(cfg, v.device)
    n = v.shape[0]
    require(v, "ind", torch.float32, (n, ctx.H, ctx.W), ctx.device)
    contact = torch.empty((n, 8), dtype=torch.float64, device=v.device)
    summary = torch.empty((n, 8), dtype=torch.float32, device=v.device)
    kind = _lib.TAC_INPUT_INDENTATION if input_kind == "indentation" else _lib.TAC_INPUT_DEPTH
    _lib.check(
        ctx.lib.tac_contact(ctx.handle, v.data_ptr(), kind, contact.data_ptr(), summary.data_ptr(),
                            ctx.workspace(n).data_ptr(), n, ctx.stream()),
        "tac_contact",
    )
    return (contact[0], summary[0]) if single else (contact, summary)


def threshold_invalid(t):
    return not (t > 0)


def track_load(prev: torch.Tensor, pose_delta: torch.Tensor, contact: torch.Tensor, cfg: PipelineConfig):
    """REF/marker.py:124-140, batched; returns the new state (prev is not modified)."""
    ctx = context_for(cfg, prev.device)
    n = prev.shape[0]
    state = prev.clone()
    require(state, "prev", torch.float64, (n, 8), ctx.device)
    require(pose_delta, "pose_delta", torch.float64, (n, 3), ctx.device)
    require(contact, "contact", torch.float64, (n, 8), ctx.device)
    _lib.check(ctx.lib.tac_track_load(ctx.handle, state.data_ptr(), pose_delta.data_ptr(),
                                      contact.data_ptr(), n, ctx.stream()), "tac_track_load")
    return state


def marker_displacements(loads: torch.Tensor, cfg: PipelineConfig) -> torch.Tensor:
    """u = u_n + u_s + u_t per marker, REF/marker.py:143-165 -> [N, rows, cols, 2] fp32."""
    ctx = context_for(cfg, loads.device)
    n = loads.shape[0]
    require(loads, "loads", torch.float64, (n, 8), ctx.device)
    disp = torch.empty((n, ctx.rows, ctx.cols, 2), dtype=torch.float32, device=loads.device)
    _lib.check(ctx.lib.tac_marker_displacements(ctx.handle, loads.data_ptr(), disp.data_ptr(), n,
                                                ctx.stream()), "tac_marker_displacements")
    return disp


def render_markers(disp: torch.Tensor, rgb: torch.Tensor, cfg: PipelineConfig) -> torch.Tensor:
    """Dot splat of REF/marker.py:203-234 (no arrows) into ``rgb`` in place."""
    ctx = context_for(cfg, disp.device)
    n = disp.shape[0]
    require(disp, "disp", torch.float32, (n, ctx.rows, ctx.cols, 2), ctx.device)
    require(rgb, "rgb", torch.uint8, (n, ctx.H, ctx.W, 3), ctx.device)
    _lib.check(ctx.lib.tac_render_markers(ctx.handle, disp.data_ptr(), rgb.data_ptr(), n,
                                          ctx.stream()), "tac_render_markers")
    return rgb
