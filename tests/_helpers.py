"""Shared test helpers: seeded inputs and oracle expectations."""

import numpy as np
import torch

from oracle import marker as omk
from oracle import pipeline as opl
from paper_2411_04776_b200 import synthetic
from paper_2411_04776_b200.config import MarkerParams, PipelineConfig, SensorConfig, levels_from_sigmas


def small_config(h=48, w=64, grid=(5, 7), sigmas=(1.0, 2.0, 4.0), seed=0, bins=(125, 180),
                 lambda_n=0.8e-3, dot_radius=3, pitch=synthetic.PITCH, levels=None, shadows=False):
    return PipelineConfig(
        sensor=SensorConfig.from_pitch(h, w, pitch, synthetic.REST, grid),
        levels=levels if levels is not None else levels_from_sigmas(sigmas),
        lut=synthetic.random_lut(seed + 1, *bins),
        background=synthetic.random_background(seed + 2, h, w),
        g_max=1.0,
        marker_params=MarkerParams(lambda_n=lambda_n),
        dot_radius=dot_radius,
        light_dirs=DEFAULT_LIGHT_DIRS if shadows else None,
        shadow_factor=0.6 if shadows else 1.0,
    )


# tacsim default_lighting() directions (REF/optical.py:68-79): R, G, B lights
# 120 degrees apart in azimuth at 35 degrees elevation, normalised as
# LightingModel does (REF/optical.py:36-45).
def _default_dirs():
    el = np.deg2rad(35.0)
    az = np.deg2rad([0.0, 120.0, 240.0])
    d = np.stack([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.full(3, np.sin(el))], axis=1)
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


DEFAULT_LIGHT_DIRS = _default_dirs()


def depth_batch(n, h, w, seed, pitch=synthetic.PITCH, **kw):
    """Seeded fp32 depth maps (generated in fp64 on the CPU, then rounded)."""
    p = synthetic.indenters(n, h, w, seed, pitch=pitch, **kw)
    return synthetic.height_maps(p, h, w, pitch=pitch, device="cpu", dtype=torch.float64).float()


def oracle_env(cfg: PipelineConfig, depth_f32, shear, twist, splat=True):
    mp = cfg.marker_params
    return opl.simulate_env(
        depth_f32.astype(np.float64),
        pitch=cfg.pixel_pitch,
        rest=cfg.sensor.gelpad_thickness,
        levels=cfg.levels,
        lut=cfg.lut.astype(np.float64),
        background=cfg.background.astype(np.float64),
        g_max=cfg.g_max,
        rest_grid=cfg.rest_grid,
        shear=shear,
        twist=twist,
        params=(mp.k_n, mp.lambda_n, mp.lambda_s, mp.k_t, mp.lambda_t),
        threshold=cfg.contact_threshold,
        dot_radius=cfg.dot_radius,
        dot_color=cfg.dot_color,
        splat=splat,
        light_dirs=cfg.light_dirs,
        shadow_factor=cfg.shadow_factor,
        shadow_steps=cfg.shadow_steps,
        shadow_softness=cfg.shadow_softness,
    )


def normwise(got, ref):
    """||got - ref||_inf / ||ref||_inf (0 when both vanish)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max() if ref.size else 0.0
    num = np.abs(got - ref).max() if ref.size else 0.0
    if den == 0.0:
        return num
    return num / den


def rgb_stats(got, ref):
    d = np.abs(got.astype(np.int32) - ref.astype(np.int32))
    return d.max() if d.size else 0, float((d <= 1).mean()) if d.size else 1.0


__all__ = ["small_config", "depth_batch", "oracle_env", "normwise", "rgb_stats", "omk"]
