"""Vectorised CPU port of the path, used only as the timed CPU baseline
(bench.py ``cpu_baseline`` and ``--impl reference``).  TEST INFRASTRUCTURE.

Same algorithm as ``oracle.pipeline.simulate_env`` but written the way the
reference itself runs it: the pyramid is ``scipy.ndimage.gaussian_filter(...,
mode="nearest", truncate=r/sigma)`` exactly as REF/tactile.py:219-221, the
gradient is ``np.gradient`` as REF/optical.py:160, and the per-pixel LUT
evaluation is one gather + fused multiply over all pixels.  float64 like the
reference.  ``tests/test_oracle_fast.py`` checks it against the oracle.
"""

import numpy as np
from scipy import ndimage

from . import marker, optical


class FastOracle:
    def __init__(self, cfg):
        self.cfg = cfg
        self.pitch = cfg.pixel_pitch
        self.rest = cfg.sensor.gelpad_thickness
        self.levels = cfg.levels
        lut = np.asarray(cfg.lut, dtype=np.float64)
        self.n_mag, self.n_dir = lut.shape[:2]
        self.lut = lut[:, :, :, 1:].reshape(self.n_mag * self.n_dir, 3, 5)
        self.bg = np.asarray(cfg.background, dtype=np.float64)
        self.g_max = cfg.g_max
        self.grid = np.asarray(cfg.rest_grid, dtype=np.float64)
        mp = cfg.marker_params
        self.params = (mp.k_n, mp.lambda_n, mp.lambda_s, mp.k_t, mp.lambda_t)
        r = cfg.dot_radius
        dy, dx = np.mgrid[-r : r + 1, -r : r + 1]
        m = dx * dx + dy * dy <= r * r
        self.sten = (dy[m], dx[m])
        self.color = np.asarray(cfg.dot_color, dtype=np.uint8)
        self.threshold = cfg.contact_threshold
        self.shadows = bool(getattr(cfg, "shadows", False))
        if self.shadows:
            self.light_dirs = np.asarray(cfg.light_dirs, dtype=np.float64)
            self.shadow_args = (cfg.shadow_factor, cfg.shadow_steps, cfg.shadow_softness)

    def run(self, depth, shear, twist):
        ind = np.clip(self.rest - depth, 0.0, self.rest)
        acc = np.zeros_like(ind)
        for sigma, r in self.levels:
            if r == 0:
                acc += ind
            else:
                acc += ndimage.gaussian_filter(ind, sigma=sigma, mode="nearest", truncate=r / sigma)
        blurred = acc / len(self.levels)
        gy, gx = np.gradient(blurred, self.pitch)
        norm = np.sqrt(gx * gx + gy * gy + 1.0)
        nx, ny = -gx / norm, -gy / norm
        gm = np.sqrt(gx * gx + gy * gy)
        mb = np.minimum(np.floor(gm / self.g_max * self.n_mag), self.n_mag - 1).astype(np.int64)
        db = np.mod(np.floor((np.arctan2(gy, gx) + np.pi) / (2 * np.pi) * self.n_dir).astype(np.int64),
                    self.n_dir)
        coef = self.lut[mb * self.n_dir + db]  # (H, W, 3, 5)
        basis = np.stack([nx, ny, nx * nx, nx * ny, ny * ny], axis=-1)
        delta = np.einsum("hwck,hwk->hwc", coef, basis)
        val = self.bg + delta
        if self.shadows:  # add_shadows (REF/optical.py:261-300) on the clipped shading
            f, steps, soft = self.shadow_args
            sh = optical.shadow_factor(-depth, self.pitch, self.light_dirs, f, steps, soft)
            val = np.clip(val, 0.0, 255.0) * sh[..., None]
        rgb = np.clip(np.rint(val), 0, 255).astype(np.uint8)
        c = marker.contact_center(ind, self.pitch, self.threshold)
        load = dict(c)
        if c["in_contact"]:
            load.update(sx=float(shear[0]), sy=float(shear[1]), twist=float(twist))
        else:
            load.update(sx=0.0, sy=0.0, twist=0.0)
        disp = marker.marker_displacements(load, self.grid, self.params)
        h, w = ind.shape
        cols, rows = marker.dot_centres(self.grid + disp, self.pitch, h, w)
        yy = (rows[:, None] + self.sten[0][None]).ravel()
        xx = (cols[:, None] + self.sten[1][None]).ravel()
        ok = (yy >= 0) & (yy < h) & (xx >= 0) & (xx < w)
        rgb[yy[ok], xx[ok]] = self.color
        return rgb, disp, marker.contact_summary(c, self.pitch), blurred
