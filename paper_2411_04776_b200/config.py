"""Configuration types mirroring the reference dataclasses.

``SensorConfig`` mirrors REF/tactile.py:31-69, ``MarkerParams`` mirrors
REF/marker.py:25-40 (same defaults, same validation, same error class).
``PipelineConfig`` is the frozen bundle uploaded once into a C-ABI context.
"""

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np

from .errors import InvalidArgumentError

DEFAULT_PYRAMID = (5, 11, 21, 31)  # REF/tactile.py:22
DEFAULT_CONTACT_THRESHOLD = 5e-5  # REF/marker.py:22


_IDENTITY_POSE = tuple(float(v) for v in np.eye(4).ravel())


@dataclass(frozen=True)
class SensorConfig:
    """Geometry of one tactile sensor (REF/tactile.py:31-69).

    ``camera_pose_in_case``: the camera frame in the sensor case frame
    (REF/tactile.py:47, used as ``case_pose.compose(camera_pose_in_case)`` at
    REF/envs.py:733-734), here a 4x4 homogeneous rigid transform stored as
    16 row-major floats (any 4x4 array-like is accepted); identity by default.
    """

    image_size: Tuple[int, int] = (480, 640)
    sensing_area: Tuple[float, float] = (0.016, 0.012)
    gelpad_thickness: float = 0.004
    marker_grid: Tuple[int, int] = (10, 10)
    camera_pose_in_case: Tuple[float, ...] = _IDENTITY_POSE

    def __post_init__(self):
        h, w = self.image_size
        if int(h) <= 0 or int(w) <= 0:
            raise InvalidArgumentError("image_size must be positive")
        aw, ah = self.sensing_area
        if aw <= 0 or ah <= 0:
            raise InvalidArgumentError("sensing_area must be positive")
        if self.gelpad_thickness <= 0:
            raise InvalidArgumentError("gelpad_thickness must be positive")
        if int(self.marker_grid[0]) <= 0 or int(self.marker_grid[1]) <= 0:
            raise InvalidArgumentError("marker_grid must be positive")
        if abs(aw / w - ah / h) > 1e-12:
            raise InvalidArgumentError("sensing_area and image_size imply unequal x/y pixel pitch")
        t = np.asarray(self.camera_pose_in_case, dtype=np.float64).reshape(-1)
        if t.size != 16 or not np.isfinite(t).all():
            raise InvalidArgumentError("camera_pose_in_case must be a finite 4x4 transform")
        m = t.reshape(4, 4)
        if not np.allclose(m[3], [0, 0, 0, 1]) or not np.allclose(m[:3, :3] @ m[:3, :3].T, np.eye(3), atol=1e-9):
            raise InvalidArgumentError("camera_pose_in_case must be a rigid transform (orthonormal rotation)")
        object.__setattr__(self, "camera_pose_in_case", tuple(float(v) for v in t))

    @property
    def camera_pose_matrix(self) -> np.ndarray:
        """camera_pose_in_case as a 4x4 float64 array."""
        return np.asarray(self.camera_pose_in_case, dtype=np.float64).reshape(4, 4)

    @property
    def pixel_pitch(self) -> float:
        return self.sensing_area[0] / self.image_size[1]

    @staticmethod
    def from_pitch(h, w, pitch, gelpad_thickness=0.004, marker_grid=(10, 10)):
        return SensorConfig((int(h), int(w)), (w * pitch, h * pitch), gelpad_thickness, marker_grid)


@dataclass(frozen=True)
class MarkerParams:
    """Displacement-distribution constants, metres (REF/marker.py:25-40)."""

    k_n: float = 0.3
    lambda_n: float = 4e-3
    lambda_s: float = 5e-3
    k_t: float = 0.5
    lambda_t: float = 4e-3

    def __post_init__(self):
        vals = (self.k_n, self.lambda_n, self.lambda_s, self.k_t, self.lambda_t)
        if not all(math.isfinite(v) for v in vals):
            raise InvalidArgumentError("marker params must be finite")
        if self.lambda_n <= 0 or self.lambda_s <= 0 or self.lambda_t <= 0:
            raise InvalidArgumentError("marker length scales must be positive")


def levels_from_kernel_sizes(kernel_sizes: Sequence[int] = DEFAULT_PYRAMID):
    """(sigma, radius) per level, REF/tactile.py:204-218 (same validation)."""
    sizes = [int(k) for k in kernel_sizes]
    if not sizes:
        raise InvalidArgumentError("kernel_sizes must be nonempty")
    for k in sizes:
        if k < 1 or k % 2 == 0:
            raise InvalidArgumentError("kernel sizes must be odd and >= 1")
    if sizes != sorted(sizes):
        raise InvalidArgumentError("kernel sizes must be ascending")
    return tuple((0.0, 0) if k == 1 else (k / 6.0, (k - 1) // 2) for k in sizes)


def levels_from_sigmas(sigmas: Sequence[float], truncate: float = 3.0):
    """(sigma, radius = ceil(truncate * sigma)) per level: the north star's
    sigma-keyed pyramid.  sigma 0 = identity level."""
    out = []
    if not len(sigmas):
        raise InvalidArgumentError("sigmas must be nonempty")
    for s in sigmas:
        s = float(s)
        if not math.isfinite(s) or s < 0:
            raise InvalidArgumentError("sigma must be finite and >= 0")
        out.append((0.0, 0) if s == 0 else (s, int(math.ceil(truncate * s - 1e-12))))
    return tuple(out)


def grid_rest_positions(cfg: SensorConfig) -> np.ndarray:
    """(rows, cols, 2) marker rest grid, REF/marker.py:93-100."""
    rows, cols = int(cfg.marker_grid[0]), int(cfg.marker_grid[1])
    w, h = cfg.sensing_area
    xs = ((np.arange(cols) + 0.5) / cols - 0.5) * w
    ys = ((np.arange(rows) + 0.5) / rows - 0.5) * h
    gx, gy = np.meshgrid(xs, ys)
    return np.stack([gx, gy], axis=-1)


@dataclass(frozen=True, eq=False)
class PipelineConfig:
    """Everything the sm_100a path needs, uploaded once per context.

    lut: (mag_bins, dir_bins, 3, 6) float32, 8-bit units, basis order of
    REF/optical.py:82-88 (c0 ignored: it cancels, REF/optical.py:244).
    background: (H, W, 3) float32 in 8-bit units.
    """

    sensor: SensorConfig
    levels: Tuple[Tuple[float, int], ...]
    lut: np.ndarray
    background: np.ndarray
    g_max: float = 1.0
    marker_params: MarkerParams = field(default_factory=MarkerParams)
    contact_threshold: float = DEFAULT_CONTACT_THRESHOLD
    dot_radius: int = 3
    dot_color: Tuple[int, int, int] = (25, 25, 25)
    rest_grid: Optional[np.ndarray] = None
    # add_shadows (REF/optical.py:261-300); factor 1.0 = off (the parity setting)
    light_dirs: Optional[np.ndarray] = None  # (n_lights, 3), e.g. default_lighting().directions
    shadow_factor: float = 1.0
    shadow_steps: int = 80
    shadow_softness: float = 5e-5
    # execution choices (tac_config.lut_dtype / kernel_path / chunk_envs):
    # lut_dtype "f16" stores the LUT coefficients in fp16 (half the shade
    # kernel's gather bytes, <= 2^-11 relative per coefficient); kernel_path
    # "auto" | "stream" | "band" | "fused" picks the tac_pipeline kernels (A/B and tests)
    lut_dtype: str = "f32"
    kernel_path: str = "auto"
    chunk_envs: int = 0

    def __post_init__(self):
        h, w = self.sensor.image_size
        lut = np.ascontiguousarray(self.lut, dtype=np.float32)
        bg = np.ascontiguousarray(self.background, dtype=np.float32)
        if lut.ndim != 4 or lut.shape[2:] != (3, 6):
            raise InvalidArgumentError("lut must be (mag_bins, dir_bins, 3, 6)")
        if bg.shape != (h, w, 3):
            raise InvalidArgumentError("background must be (H, W, 3)")
        if not (np.isfinite(lut).all() and np.isfinite(bg).all()):
            raise InvalidArgumentError("table values must be finite")
        if not (self.g_max > 0 and math.isfinite(self.g_max)):
            raise InvalidArgumentError("g_max must be positive")
        if self.contact_threshold <= 0:
            raise InvalidArgumentError("threshold must be positive")
        if not self.levels:
            raise InvalidArgumentError("pyramid needs at least one level")
        object.__setattr__(self, "lut", lut)
        object.__setattr__(self, "background", bg)
        grid = self.rest_grid
        if grid is None:
            grid = grid_rest_positions(self.sensor)
        grid = np.ascontiguousarray(grid, dtype=np.float64)
        if grid.shape != (self.sensor.marker_grid[0], self.sensor.marker_grid[1], 2):
            raise InvalidArgumentError("rest_positions must be (rows, cols, 2)")
        object.__setattr__(self, "rest_grid", grid)
        if not 0.0 <= self.shadow_factor <= 1.0:
            raise InvalidArgumentError("shadow factor must be in [0, 1]")
        dirs = np.zeros((0, 3)) if self.light_dirs is None else np.asarray(self.light_dirs, np.float64)
        if dirs.ndim != 2 or dirs.shape[1] != 3 or len(dirs) > 4:
            raise InvalidArgumentError("light_dirs must be (n <= 4, 3)")
        object.__setattr__(self, "light_dirs", dirs)
        if self.lut_dtype not in ("f32", "f16"):
            raise InvalidArgumentError("lut_dtype must be 'f32' or 'f16'")
        if self.kernel_path not in ("auto", "stream", "band", "fused"):
            raise InvalidArgumentError("kernel_path must be 'auto', 'stream', 'band' or 'fused'")
        if int(self.chunk_envs) < 0:
            raise InvalidArgumentError("chunk_envs must be >= 0")

    @property
    def shadows(self) -> bool:
        return self.shadow_factor != 1.0 and len(self.light_dirs) > 0

    @property
    def pixel_pitch(self):
        return self.sensor.pixel_pitch
