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
