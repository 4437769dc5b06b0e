"""Oracle: contact centroid, load tracking, marker field, dot splat
(TEST INFRASTRUCTURE).

float64 NumPy restatement of ``tacsim/marker.py``.  Loads are plain dicts /
arrays instead of the reference dataclasses so batches are cheap.
"""

import numpy as np

# marker.py:22
DEFAULT_CONTACT_THRESHOLD = 5e-5

# marker.py:29-33 (k_n, lambda_n, lambda_s, k_t, lambda_t)
DEFAULT_PARAMS = (0.3, 4e-3, 5e-3, 0.5, 4e-3)


def grid_rest_positions(rows, cols, area_w, area_h):
    """(rows, cols, 2) marker rest grid centred on the sensing area.

    marker.py:93-100: x_j = ((j + 0.5)/cols - 0.5) * w, y_i likewise.
    """
    xs = ((np.arange(cols) + 0.5) / cols - 0.5) * area_w
    ys = ((np.arange(rows) + 0.5) / rows - 0.5) * area_h
    gx, gy = np.meshgrid(xs, ys)
    return np.stack([gx, gy], axis=-1)


def contact_center(ind, pitch, threshold=DEFAULT_CONTACT_THRESHOLD):
    """Indentation-weighted centroid of pixels with ind > threshold.

    marker.py:103-121: strict '>' mask; weights = raw indentation; pixel
    centres (j + 0.5 - W/2) * p, (i + 0.5 - H/2) * p; d_c = max over the whole
    map; all zero when no pixel passes.  Returns a dict with the load fields
    plus the builder-defined summary terms (count, weight sum).
    """
    vals = np.asarray(ind, dtype=np.float64)
    if threshold <= 0:
        raise ValueError("threshold must be positive")
    mask = vals > threshold
    if not mask.any():
        return dict(cx=0.0, cy=0.0, dmax=0.0, in_contact=False, count=0, wsum=0.0)
    h, w = vals.shape
    ii, jj = np.nonzero(mask)
    weights = vals[ii, jj]
    xs = (jj + 0.5 - 0.5 * w) * pitch
    ys = (ii + 0.5 - 0.5 * h) * pitch
    total = weights.sum()
    return dict(
        cx=float((weights * xs).sum() / total),
        cy=float((weights * ys).sum() / total),
        dmax=float(vals.max()),
        in_contact=True,
        count=int(mask.sum()),
        wsum=float(total),
    )


def contact_summary(load, pitch):
    """Builder-defined per-env summary, 8 values:
    [in_contact, area = count*p^2, c_x, c_y, d_c, force proxy = sum(ind)*p^2
    over the contact mask, 0, 0]."""
    return np.array(
        [
            1.0 if load["in_contact"] else 0.0,
            load["count"] * pitch * pitch,
            load["cx"],
            load["cy"],
            load["dmax"],
            load["wsum"] * pitch * pitch,
            0.0,
            0.0,
        ]
    )


def track_load(prev, delta, contact):
    """Advance accumulated shear / twist by one case-pose delta.

    marker.py:124-140.  ``prev`` and the result are dicts with keys cx, cy,
    dmax, sx, sy, twist, in_contact; ``delta`` = (dx, dy, rotvec_z) of the
    case pose delta; ``contact`` is a ``contact_center`` result.
    """
    if not contact["in_contact"]:
        return dict(cx=0.0, cy=0.0, dmax=0.0, sx=0.0, sy=0.0, twist=0.0, in_contact=False)
    out = dict(cx=contact["cx"], cy=contact["cy"], dmax=contact["dmax"], in_contact=True)
    if not prev["in_contact"]:
        out.update(sx=0.0, sy=0.0, twist=0.0)
        return out
    out.update(
        sx=prev["sx"] + float(delta[0]),
        sy=prev["sy"] + float(delta[1]),
        twist=prev["twist"] - float(delta[2]),
    )
    return out


def marker_displacements(load, rest, params=DEFAULT_PARAMS):
    """u = u_n + u_s + u_t per marker.  marker.py:143-165.

    ``load`` needs cx, cy, dmax, sx, sy, twist, in_contact.
    """
    k_n, lam_n, lam_s, k_t, lam_t = params
    rest = np.asarray(rest, dtype=np.float64)
    if not load["in_contact"]:
        return np.zeros_like(rest)
    c = np.array([load["cx"], load["cy"]])
    r = rest - c
    dist = np.linalg.norm(r, axis=-1)
    safe = np.where(dist > 0, dist, 1.0)
    radial = r / safe[..., None]
    u_n = (k_n * load["dmax"] * np.exp(-dist / lam_n))[..., None] * radial
    u_n[dist == 0] = 0.0
    s = np.array([load["sx"], load["sy"]])
    u_s = np.exp(-(dist * dist) / (2 * lam_s**2))[..., None] * s
    perp = np.stack([-r[..., 1], r[..., 0]], axis=-1)
    u_t = (load["twist"] * k_t * np.exp(-dist / lam_t))[..., None] * perp
    return u_n + u_s + u_t


def dot_centres(positions, pitch, h, w):
    """Integer dot centres (col, row) = round(p/pitch + W/2 - 0.5), Python
    round (half-to-even).  marker.py:221-225."""
    p = np.asarray(positions, dtype=np.float64).reshape(-1, 2)
    cols = np.round(p[:, 0] / pitch + 0.5 * w - 0.5).astype(np.int64)
    rows = np.round(p[:, 1] / pitch + 0.5 * h - 0.5).astype(np.int64)
    return cols, rows


def render_markers(img_u8, positions, pitch, radius=4, color=(25, 25, 25)):
    """Splat filled dots into a copy of ``img_u8`` (H, W, 3).

    marker.py:227-233 draws ``cv2.circle(img, c, r, color, -1)`` for each
    marker; for integer centres that pixel set is exactly
    {dx^2 + dy^2 <= r^2} clipped to the image (verified against cv2 for
    r = 0..12 in tests/golden/make_golden.py).
    """
    img = np.array(img_u8, dtype=np.uint8, copy=True)
    h, w = img.shape[:2]
    cols, rows = dot_centres(positions, pitch, h, w)
    col = np.asarray(color, dtype=np.uint8)
    for cx, cy in zip(cols, rows):
        for dy in range(-radius, radius + 1):
            y = cy + dy
            if y < 0 or y >= h:
                continue
            for dx in range(-radius, radius + 1):
                x = cx + dx
                if 0 <= x < w and dx * dx + dy * dy <= radius * radius:
                    img[y, x] = col
    return img
