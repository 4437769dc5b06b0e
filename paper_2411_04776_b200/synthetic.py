"""Seeded synthetic workloads of BASELINE.json configs[0..4].

BASELINE names no public dataset: these generators are the workload
(SURVEY.md §8(d)).  Height maps are depth-from-camera maps (HeightMap
semantics, REF/tactile.py:3-8): depth = rest - penetration profile.

Primitive choices the configs leave open (documented in DESIGN.md §6):
sphere radius 4 mm; cylinder radius 3 mm (line contact, random yaw); cube
edge = a 90-degree edge pressed point-first (faces at 45 degrees, slope 1,
random yaw); plate = flat plate at penetration d textured with 2-D Perlin
gradient noise of amplitude 0.05 mm and 1 mm lattice (random offset/yaw).
Centres are uniform in the middle 50% of each axis.
"""

import math
from dataclasses import dataclass

import numpy as np
import torch

from .config import MarkerParams, PipelineConfig, SensorConfig, levels_from_sigmas

PITCH = 0.0266e-3  # m / px (configs: 0.0266 mm/px)
REST = 4e-3  # gel thickness, REF/tactile.py:45
KINDS = ("sphere", "cylinder", "edge", "perlin")


@dataclass
class IndenterParams:
    kind: np.ndarray  # [N] int (index into KINDS)
    pen: np.ndarray  # [N] penetration, m
    cx: np.ndarray  # [N] centre, m (sensor frame)
    cy: np.ndarray
    yaw: np.ndarray  # [N] rad
    perm: np.ndarray  # [N, 256] Perlin permutation
    off: np.ndarray  # [N, 2] Perlin lattice offset

    def subset(self, idx):
        """The indenters of the given env indices (a slice or an index array)."""
        return IndenterParams(*(getattr(self, f)[idx] for f in ("kind", "pen", "cx", "cy", "yaw", "perm", "off")))


def indenters(n, h, w, seed, *, kinds=KINDS, pen=(0.0, 1.2e-3), pitch=PITCH, fixed_kind=None):
    rng = np.random.default_rng(seed)
    if fixed_kind:
        kind = np.full(n, KINDS.index(fixed_kind))
    else:
        kind = np.array([KINDS.index(kinds[i % len(kinds)]) for i in range(n)], dtype=np.int64)
    if np.isscalar(pen):
        p = np.full(n, float(pen))
    else:
        p = rng.uniform(pen[0], pen[1], n)
    ax, ay = w * pitch, h * pitch
    cx = rng.uniform(-0.25 * ax, 0.25 * ax, n)
    cy = rng.uniform(-0.25 * ay, 0.25 * ay, n)
    yaw = rng.uniform(0.0, 2 * math.pi, n)
    perm = np.stack([rng.permutation(256) for _ in range(n)])
    off = rng.uniform(0.0, 256.0, (n, 2))
    return IndenterParams(kind, p, cx, cy, yaw, perm, off)


def _fade(t):
    return t * t * t * (t * (t * 6.0 - 15.0) + 10.0)


def _perlin(u, v, perm):
    """2-D gradient noise in about [-1, 1].  u, v: [n, H, W]; perm: [n, 256] long."""
    i0 = torch.floor(u)
    j0 = torch.floor(v)
    fu, fv = u - i0, v - j0
    i0 = i0.long()
    j0 = j0.long()
    n = u.shape[0]
    flat = perm.reshape(n, 256)

    def grad_dot(di, dj):
        ii = (i0 + di) & 255
        jj = (j0 + dj) & 255
        a = torch.gather(flat, 1, ii.reshape(n, -1)).reshape(ii.shape)
        hsh = torch.gather(flat, 1, ((a + jj) & 255).reshape(n, -1)).reshape(ii.shape)
        ang = hsh.to(u.dtype) * (2 * math.pi / 256.0)
        return torch.cos(ang) * (fu - di) + torch.sin(ang) * (fv - dj)

    su, sv = _fade(fu), _fade(fv)
    n00, n10, n01, n11 = grad_dot(0, 0), grad_dot(1, 0), grad_dot(0, 1), grad_dot(1, 1)
    nx0 = n00 + su * (n10 - n00)
    nx1 = n01 + su * (n11 - n01)
    return math.sqrt(2.0) * (nx0 + sv * (nx1 - nx0))


def height_maps(params: IndenterParams, h, w, *, pitch=PITCH, rest=REST, device="cpu",
                dtype=torch.float64, chunk=256, out=None, out_dtype=torch.float32):
    """Depth maps [N, H, W] for the given indenters (computed in ``dtype``)."""
    n = len(params.kind)
    if out is None:
        out = torch.empty((n, h, w), dtype=out_dtype, device=device)
    ys = (torch.arange(h, device=device, dtype=dtype) + 0.5 - 0.5 * h) * pitch
    xs = (torch.arange(w, device=device, dtype=dtype) + 0.5 - 0.5 * w) * pitch
    gy, gx = torch.meshgrid(ys, xs, indexing="ij")
    t = lambda a: torch.as_tensor(a, device=device, dtype=dtype)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        kind = torch.as_tensor(params.kind[s:e], device=device)
        pen = t(params.pen[s:e])[:, None, None]
        dx = gx[None] - t(params.cx[s:e])[:, None, None]
        dy = gy[None] - t(params.cy[s:e])[:, None, None]
        yaw = t(params.yaw[s:e])[:, None, None]
        c, sn = torch.cos(yaw), torch.sin(yaw)
        along = dx * c + dy * sn
        perp = -dx * sn + dy * c
        ind = torch.zeros((e - s, h, w), device=device, dtype=dtype)
        # sphere r = 4 mm
        r = 4e-3
        rho2 = dx * dx + dy * dy
        sph = torch.clamp(pen - r + torch.sqrt(torch.clamp(r * r - rho2, min=0.0)), min=0.0)
        sph = torch.where(rho2 < r * r, sph, torch.zeros_like(sph))
        # cylinder r = 3 mm, axis along `along`
        rc = 3e-3
        cyl = torch.clamp(pen - rc + torch.sqrt(torch.clamp(rc * rc - perp * perp, min=0.0)), min=0.0)
        cyl = torch.where(perp * perp < rc * rc, cyl, torch.zeros_like(cyl))
        # 90-degree cube edge (slope 1 faces)
        edge = torch.clamp(pen - perp.abs(), min=0.0)
        ind = torch.where((kind == 0)[:, None, None], sph, ind)
        ind = torch.where((kind == 1)[:, None, None], cyl, ind)
        ind = torch.where((kind == 2)[:, None, None], edge, ind)
        if bool((kind == 3).any()):
            cell = 1e-3
            off = t(params.off[s:e])
            u = along / cell + off[:, 0, None, None]
            v = perp / cell + off[:, 1, None, None]
            perm = torch.as_tensor(params.perm[s:e], device=device, dtype=torch.long)
            pl = torch.clamp(pen + 0.05e-3 * _perlin(u, v, perm), min=0.0)
            ind = torch.where((kind == 3)[:, None, None], pl, ind)
        out[s:e] = (rest - ind).to(out.dtype)
    return out


def random_lut(seed, mag_bins=125, dir_bins=180):
    """Seeded LUT U[-1, 1] of shape (mag, dir, 3, 6) (configs[0])."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (mag_bins, dir_bins, 3, 6)).astype(np.float32)


def random_background(seed, h, w):
    """fp32 background U[80, 160] in 8-bit units (configs[0])."""
    return np.random.default_rng(seed).uniform(80.0, 160.0, (h, w, 3)).astype(np.float32)


def loads(n, seed):
    """configs[2] loads: shear U(+-0.3 mm) per axis, twist U(+-5 deg)."""
    rng = np.random.default_rng(seed)
    shear = rng.uniform(-0.3e-3, 0.3e-3, (n, 2))
    twist = rng.uniform(-math.radians(5.0), math.radians(5.0), n)
    return shear, twist


def baseline_config(index, seed=0):
    """(PipelineConfig, n_env) for BASELINE.json configs[index]."""
    if index == 3:
        h, w, sig, grid = 480, 640, (1.0, 2.0, 4.0, 8.0), (14, 18)
    else:
        h, w, sig, grid = 240, 320, (1.0, 2.0, 4.0), (7, 9)
    n = {0: 1, 1: 1024, 2: 4096, 3: 1024, 4: 32768}[index]
    params = MarkerParams(lambda_n=0.8e-3) if index >= 2 else MarkerParams()
    cfg = PipelineConfig(
        sensor=SensorConfig.from_pitch(h, w, PITCH, REST, grid),
        levels=levels_from_sigmas(sig),
        lut=random_lut(seed + 1),
        background=random_background(seed + 2, h, w),
        g_max=1.0,
        marker_params=params,
        dot_radius=3,
    )
    return cfg, n


def workload(index, seed=0, n_total=None):
    """The seeded global workload of configs[index]: (cfg, n_total, indenter
    params of every env, shear [n,2], twist [n]).  Env e has the same frame
    and load whatever the GPU count, so ranks slice it with
    ``sharding.env_block`` (strong scaling) and the CPU baseline samples it."""
    cfg, n = baseline_config(index, seed)
    if n_total:
        n = int(n_total)
    h, w = cfg.sensor.image_size
    params = indenters(n, h, w, seed + 10)
    shear, twist = loads(n, seed + 20)
    return cfg, n, params, shear, twist
