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


def shade_lut(blurred, pitch, lut, background, g_max):
    """Binned-LUT shading of a smoothed indentation map -> uint8 RGB.

    Builder's definition (SURVEY.md Appendix "Binned-LUT definition"):
    gradient as np.gradient (optical.py:160), normals as optical.py:161-162,
    per-pixel bins (``lut_bins``), Delta_c = sum_{k=1..5} LUT[mb, db, c, k] *
    basis_k(nx, ny) with the basis order of optical.py:82-88 (c0 cancels as in
    optical.py:244), then rgb = clip(rint(bg + Delta), 0, 255) with bg in
    8-bit units.  ``lut`` is (n_mag, n_dir, 3, 6), ``background`` (H, W, 3).
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
    raw = np.rint(np.asarray(background, dtype=np.float64) + delta)
    out = np.clip(raw, 0.0, 255.0)
    return out.astype(np.uint8), int((raw != out).sum())


def lut_from_global(coeffs, n_mag, n_dir, scale=255.0):
    """Fill every bin with the global table (8-bit units): the degenerate
    LUT under which ``shade_lut`` reproduces reference ``shade`` + uint8 rule
    to within 1 LSB (the only reference anchor of the binned LUT)."""
    c = np.asarray(coeffs, dtype=np.float64) * scale
    return np.broadcast_to(c, (n_mag, n_dir) + c.shape).copy()
