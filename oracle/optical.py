"""Oracle: gradient, normals, polynomial / binned-LUT shading (TEST INFRASTRUCTURE).

float64 NumPy restatement of ``tacsim/optical.py`` plus this repo's
definition of the north star's binned LUT (no reference implementation
exists: the reference deliberately evaluates one global polynomial,
``REF/SPEC.md:449``).
"""

import numpy as np


def gradient(elev, pitch):
    """(gy, gx) of an elevation field, as ``np.gradient(elev, pitch)``.

    Restates the call at optical.py:160: central differences
    (f[i+1]-f[i-1])/(2p) inside, one-sided first-order differences
    (f[1]-f[0])/p and (f[n-1]-f[n-2])/p on the borders.  Axis -2 -> gy,
    axis -1 -> gx.  Needs at least 2 samples per axis.
    """
    e = np.asarray(elev, dtype=np.float64)
    if e.shape[-1] < 2 or e.shape[-2] < 2:
        raise ValueError("gradient needs at least 2 samples per axis")

    def d(a, axis):
        n = a.shape[axis]
        g = np.empty_like(a)
        sl = lambda s: tuple(
            [slice(None)] * (a.ndim + axis) + [s] + [slice(None)] * (-axis - 1)
        )
        g[sl(slice(1, n - 1))] = (a[sl(slice(2, n))] - a[sl(slice(0, n - 2))]) / (2.0 * pitch)
        g[sl(0)] = (a[sl(1)] - a[sl(0)]) / pitch
        g[sl(n - 1)] = (a[sl(n - 1)] - a[sl(n - 2)]) / pitch
        return g

    return d(e, -2), d(e, -1)


def normals_from(elev, pitch):
    """Unit normals (..., H, W, 3) = (-gx, -gy, 1)/norm.  optical.py:159-163.

    ``elev`` is an elevation field (an IndentationMap's values; a HeightMap
    would be negated first, optical.py:147-149).
    """
    gy, gx = gradient(elev, pitch)
    n = np.stack([-gx, -gy, np.ones_like(gx)], axis=-1)
    n /= np.linalg.norm(n, axis=-1, keepdims=True)
    return n


def poly_exponents(degree=2):
    """Monomial order 1, x, y, x^2, xy, y^2, ...  optical.py:82-88."""
    out = []
    for total in range(degree + 1):
        for ix in range(total, -1, -1):
            out.append((ix, total - ix))
    return tuple(out)


def poly_basis(nx, ny, degree=2):
    """Stacked monomials (..., n_terms).  optical.py:91-94."""
    return np.stack(
        [np.power(nx, ix) * np.power(ny, iy) for ix, iy in poly_exponents(degree)],
        axis=-1,
    )


def shade_global(normals, coeffs, background):
    """Reference global-table shading, float in [0, 1].  optical.py:233-250.

    out = clip(bg + P(nx, ny) - c0, 0, 1) with P the per-channel polynomial
    (coeffs (3, n_terms)).  Returns (out, saturated_fraction).
    """
    n = np.asarray(normals, dtype=np.float64)
    c = np.asarray(coeffs, dtype=np.float64)
    degree = {3: 1, 6: 2, 10: 3}[c.shape[1]]
    delta = poly_basis(n[..., 0], n[..., 1], degree) @ c.T - c[:, 0]
    raw = background + delta
    out = np.clip(raw, 0.0, 1.0)
    return out, float((raw != out).mean())


def quantize_u8(x01):
    """np.round(np.clip(x, 0, 1) * 255) as uint8 (half-to-even).

    cli.py:134-139 and marker.py:219.
    """
    return np.round(np.clip(x01, 0.0, 1.0) * 255.0).astype(np.uint8)


def lut_bins(gx, gy, g_max, n_mag, n_dir):
    """Builder-defined bin indices of the binned LUT.

    magnitude bin = min(floor(|g| / g_max * n_mag), n_mag - 1)
    direction bin = floor((atan2(gy, gx) + pi) / (2 pi) * n_dir) mod n_dir
    """
    gm = np.sqrt(gx * gx + gy * gy)
    mb = np.minimum(np.floor(gm / g_max * n_mag), n_mag - 1).astype(np.int64)
    db = np.floor((np.arctan2(gy, gx) + np.pi) / (2.0 * np.pi) * n_dir).astype(np.int64)
    db = np.mod(db, n_dir)
    return mb, db


def shade_lut(blurred, pitch, lut, background, g_max, shadow=None):
    """Binned-LUT shading of a smoothed indentation map -> uint8 RGB.

    Builder's definition (SURVEY.md Appendix "Binned-LUT definition"):
    gradient as np.gradient (optical.py:160), normals as optical.py:161-162,
    per-pixel bins (``lut_bins``), Delta_c = sum_{k=1..5} LUT[mb, db, c, k] *
    basis_k(nx, ny) with the basis order of optical.py:82-88 (c0 cancels as in
    optical.py:244), then rgb = clip(rint(bg + Delta), 0, 255) with bg in
    8-bit units.  ``lut`` is (n_mag, n_dir, 3, 6), ``background`` (H, W, 3).
    With ``shadow`` (H, W) the clipped shading is multiplied by it before
    rounding (shade clips, optical.py:246; add_shadows multiplies, :299).
    Returns (rgb_u8, saturated_count).
    """
    lut = np.asarray(lut, dtype=np.float64)
    n_mag, n_dir = lut.shape[:2]
    gy, gx = gradient(blurred, pitch)
    n = np.stack([-gx, -gy, np.ones_like(gx)], axis=-1)
    n /= np.linalg.norm(n, axis=-1, keepdims=True)
    mb, db = lut_bins(gx, gy, g_max, n_mag, n_dir)
    coef = lut[mb, db]  # (..., H, W, 3, 6)
    basis = poly_basis(n[..., 0], n[..., 1], 2)  # (..., H, W, 6)
    delta = np.einsum("...ck,...k->...c", coef[..., 1:], basis[..., 1:])
    val = np.asarray(background, dtype=np.float64) + delta
    if shadow is not None:
        val = np.clip(val, 0.0, 255.0) * np.asarray(shadow, dtype=np.float64)[..., None]
    raw = np.rint(val)
    out = np.clip(raw, 0.0, 255.0)
    return out.astype(np.uint8), int((raw != out).sum())


def lut_from_global(coeffs, n_mag, n_dir, scale=255.0):
    """Fill every bin with the global table (8-bit units): the degenerate
    LUT under which ``shade_lut`` reproduces reference ``shade`` + uint8 rule
    to within 1 LSB (the only reference anchor of the binned LUT)."""
    c = np.asarray(coeffs, dtype=np.float64) * scale
    return np.broadcast_to(c, (n_mag, n_dir) + c.shape).copy()


def shadow_offsets(direction, max_steps):
    """Per-step pixel offsets (di, dj) of the march toward one light.

    optical.py:283-291: lateral = hypot(lx, ly); dx, dy = lx/lateral,
    ly/lateral; di = int(round(s*dy)), dj = int(round(s*dx)) (Python round =
    half-to-even); rise_per_px = pitch * lz / lateral.  Returns None for an
    overhead light (lateral < 1e-9), else (di[], dj[], lz / lateral).
    """
    lx, ly, lz = (float(v) for v in direction)
    lateral = float(np.hypot(lx, ly))
    if lateral < 1e-9:
        return None
    dx, dy = lx / lateral, ly / lateral
    di = np.array([int(round(s * dy)) for s in range(1, max_steps + 1)])
    dj = np.array([int(round(s * dx)) for s in range(1, max_steps + 1)])
    return di, dj, lz / lateral


def shadow_factor(elev, pitch, directions, factor=0.6, max_steps=80, softness=5e-5):
    """Multiplicative shadow factor (H, W) of add_shadows, optical.py:261-300.

    For each light: occ = max_s (elev[clip(i+di_s), clip(j+dj_s)] - elev -
    s*rise), weight = clip(occ/softness, 0, 1), and the image is multiplied by
    1 - (1 - factor) * weight; the product over lights is returned.  ``elev``
    is the elevation (a HeightMap's -values).
    """
    e = np.asarray(elev, dtype=np.float64)
    h, w = e.shape
    out = np.ones_like(e)
    if factor == 1.0:
        return out
    for d in directions:
        off = shadow_offsets(d, max_steps)
        if off is None:
            continue
        di, dj, rise = off
        rise_per_px = pitch * rise
        occ = np.full(e.shape, -np.inf)
        for s in range(max_steps):
            ii = np.clip(np.arange(h) + di[s], 0, h - 1)
            jj = np.clip(np.arange(w) + dj[s], 0, w - 1)
            np.maximum(occ, e[np.ix_(ii, jj)] - e - (s + 1) * rise_per_px, out=occ)
        out = out * (1.0 - (1.0 - factor) * np.clip(occ / softness, 0.0, 1.0))
    return out


def add_shadows(rgb, elev, pitch, directions, factor=0.6, max_steps=80, softness=5e-5):
    """rgb (H, W, 3) float times the per-light factors, applied light by light
    in the reference order (optical.py:293-299)."""
    img = np.array(rgb, dtype=np.float64, copy=True)
    if factor == 1.0:
        return img
    e = np.asarray(elev, dtype=np.float64)
    h, w = e.shape
    for d in directions:
        off = shadow_offsets(d, max_steps)
        if off is None:
            continue
        di, dj, rise = off
        rise_per_px = pitch * rise
        occ = np.full(e.shape, -np.inf)
        for s in range(max_steps):
            ii = np.clip(np.arange(h) + di[s], 0, h - 1)
            jj = np.clip(np.arange(w) + dj[s], 0, w - 1)
            np.maximum(occ, e[np.ix_(ii, jj)] - e - (s + 1) * rise_per_px, out=occ)
        img *= (1.0 - (1.0 - factor) * np.clip(occ / softness, 0.0, 1.0))[..., None]
    return img
