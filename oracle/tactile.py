"""Oracle: gel clamp and multi-scale Gaussian pyramid (TEST INFRASTRUCTURE).

float64 NumPy restatement of ``tacsim/tactile.py``.  Arrays may carry any
number of leading batch (env) dimensions; the last two axes are (H, W).
"""

import math

import numpy as np

# tactile.py:22
DEFAULT_PYRAMID = (5, 11, 21, 31)


def indentation_from(depth, rest):
    """ind = clip(rest - depth, 0, rest).  Follows tactile.py:193-197."""
    d = np.asarray(depth, dtype=np.float64)
    return np.clip(rest - d, 0.0, rest)


def levels_from_kernel_sizes(kernel_sizes=DEFAULT_PYRAMID):
    """(sigma, radius) per level from odd kernel sizes.

    Follows tactile.py:204-218: sizes must be non-empty, odd, >= 1 and
    ascending; sigma = k/6, radius = (k-1)//2; k == 1 is the identity
    (returned as sigma 0, radius 0).
    """
    sizes = [int(k) for k in kernel_sizes]
    if not sizes:
        raise ValueError("kernel_sizes must be nonempty")
    for k in sizes:
        if k < 1 or k % 2 == 0:
            raise ValueError("kernel sizes must be odd and >= 1")
    if sizes != sorted(sizes):
        raise ValueError("kernel sizes must be ascending")
    out = []
    for k in sizes:
        if k == 1:
            out.append((0.0, 0))
        else:
            out.append((k / 6.0, (k - 1) // 2))
    return out


def levels_from_sigmas(sigmas, truncate=3.0):
    """(sigma, radius) per level for the north star's sigma-parameterised
    pyramid: radius = ceil(truncate*sigma).  The reference equivalent is the
    same ``gaussian_filter(..., mode="nearest", truncate=radius/sigma)`` call
    as tactile.py:219-221 with sigma supplied directly.
    sigma == 0 is the identity level.
    """
    out = []
    for s in sigmas:
        s = float(s)
        if s < 0 or not math.isfinite(s):
            raise ValueError("sigma must be finite and >= 0")
        if s == 0.0:
            out.append((0.0, 0))
        else:
            out.append((s, int(math.ceil(truncate * s - 1e-12))))
    return out


def gaussian_weights(sigma, radius):
    """Normalised 1-D Gaussian taps for |x| <= radius.

    Restates scipy.ndimage._filters._gaussian_kernel1d (order 0), the kernel
    behind tactile.py:219: phi = exp(-0.5 x^2 / sigma^2) / sum.
    """
    if radius == 0:
        return np.ones(1)
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * x.astype(np.float64) ** 2)
    return phi / phi.sum()


def _correlate_nearest(a, w, axis):
    """1-D correlation along ``axis`` with replicate ("nearest") padding."""
    r = (len(w) - 1) // 2
    n = a.shape[axis]
    out = np.zeros_like(a)
    for t in range(-r, r + 1):
        idx = np.clip(np.arange(n) + t, 0, n - 1)
        out += w[t + r] * np.take(a, idx, axis=axis)
    return out


def gaussian_blur(ind, sigma, radius):
    """Separable blur, axis -2 (rows) then axis -1 (cols), replicate borders.

    Same operator as ``ndimage.gaussian_filter(v, sigma, mode="nearest",
    truncate=radius/sigma)`` (tactile.py:219-221), which filters axis 0 then
    axis 1 with ``correlate1d``.
    """
    a = np.asarray(ind, dtype=np.float64)
    if radius == 0:
        return a.copy()
    w = gaussian_weights(sigma, radius)
    return _correlate_nearest(_correlate_nearest(a, w, -2), w, -1)


def smooth_pyramid(ind, levels):
    """Mean over levels of the Gaussian blurs.  Follows tactile.py:212-222.

    ``levels`` is a list of (sigma, radius) from ``levels_from_kernel_sizes``
    or ``levels_from_sigmas``.
    """
    a = np.asarray(ind, dtype=np.float64)
    acc = np.zeros_like(a)
    for sigma, radius in levels:
        if radius == 0:
            acc += a
        else:
            acc += gaussian_blur(a, sigma, radius)
    return acc / len(levels)


def render_heightmap(verts_cam, tris, h, w, pitch, rest):
    """Orthographic z-buffer of camera-frame triangles (TEST INFRASTRUCTURE).

    Restates tactile.py:129-150 and the per-triangle raster of
    tactile.py:153-190 in float64: triangles whose nearest vertex is beyond
    the rest surface or whose bounding box misses the sensing window are
    culled; nearly edge-on triangles (|det| < 1e-18) are skipped; a pixel
    centre ((j + 0.5 - w/2) p, (i + 0.5 - h/2) p) is covered when all three
    barycentrics are >= -1e-12; covered hits with z <= rest lower the depth,
    which starts at rest everywhere.  The arithmetic is written in the same
    operation order as the reference so the result matches it bit for bit.
    """
    v = np.asarray(verts_cam, dtype=np.float64)
    t = np.asarray(tris, dtype=np.int64)
    depth = np.full((h, w), float(rest))
    if t.size == 0:
        return depth
    c = v[t]  # (m, 3 corners, xyz)
    hw, hh = 0.5 * w * pitch, 0.5 * h * pitch
    x, y, z = c[..., 0], c[..., 1], c[..., 2]
    live = ((z.min(1) <= rest) & (x.max(1) >= -hw) & (x.min(1) <= hw)
            & (y.max(1) >= -hh) & (y.min(1) <= hh))
    for k in np.flatnonzero(live):
        (x0, y0, z0), (x1, y1, z1), (x2, y2, z2) = c[k]
        det = (y1 - y2) * (x0 - x2) + (x2 - x1) * (y0 - y2)
        if abs(det) < 1e-18:
            continue
        lo_j = max(0, int(np.ceil(min(x0, x1, x2) / pitch + 0.5 * w - 0.5)))
        hi_j = min(w - 1, int(np.floor(max(x0, x1, x2) / pitch + 0.5 * w - 0.5)))
        lo_i = max(0, int(np.ceil(min(y0, y1, y2) / pitch + 0.5 * h - 0.5)))
        hi_i = min(h - 1, int(np.floor(max(y0, y1, y2) / pitch + 0.5 * h - 0.5)))
        if hi_j < lo_j or hi_i < lo_i:
            continue
        cx = (np.arange(lo_j, hi_j + 1) + 0.5 - 0.5 * w) * pitch
        cy = (np.arange(lo_i, hi_i + 1) + 0.5 - 0.5 * h) * pitch
        px, py = cx[None, :], cy[:, None]
        b0 = ((y1 - y2) * (px - x2) + (x2 - x1) * (py - y2)) / det
        b1 = ((y2 - y0) * (px - x2) + (x0 - x2) * (py - y2)) / det
        b2 = 1.0 - b0 - b1
        zz = b0 * z0 + b1 * z1 + b2 * z2
        ok = (b0 >= -1e-12) & (b1 >= -1e-12) & (b2 >= -1e-12) & (zz <= rest)
        win = depth[lo_i:hi_i + 1, lo_j:hi_j + 1]
        win[ok] = np.minimum(win[ok], zz[ok])
    return depth
