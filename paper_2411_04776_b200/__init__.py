"""B200-native tactile-image path (TacEx / tacsim sensing layer, arXiv 2411.04776).

Batched, drop-in mirrors of the reference sensing API (REF/__init__.py:59-81)
backed by hand-written sm_100a kernels in ``libtac_b200.so``:

* ``TactilePipeline.simulate`` — the hot path: one ``tac_pipeline`` call per
  step (band blur + shade kernels and a per-env epilogue).
* ``render_heightmap`` / ``render_heightmaps`` — the mesh -> depth z-buffer
  that feeds it (row f2).
* ``SensorObserver`` — N sensors stepped like ``Environment._observe``
  (render -> pipeline with ``track_load`` on camera-pose deltas, row f3).
* ``indentation_from``, ``smooth_pyramid`` (tactile), ``normals_from``,
  ``shade`` (optical), ``contact_center``, ``track_load``,
  ``marker_displacements``, ``render_markers`` (marker) — the individual
  reference functions, batched over a leading env dimension.
"""

from .config import (
    DEFAULT_CONTACT_THRESHOLD,
    DEFAULT_PYRAMID,
    MarkerParams,
    PipelineConfig,
    SensorConfig,
    grid_rest_positions,
    levels_from_kernel_sizes,
    levels_from_sigmas,
)
from .errors import (
    CalibrationError,
    InvalidArgumentError,
    NativeLibraryError,
    TacsimError,
    UnsupportedConfigError,
)

__version__ = "0.1.0"

_LAZY = {
    "TactilePipeline": ".pipeline",
    "Observation": ".pipeline",
    "HeightMap": ".tactile",
    "IndentationMap": ".tactile",
    "indentation_from": ".tactile",
    "smooth_pyramid": ".tactile",
    "contact_blur": ".tactile",
    "render_heightmap": ".tactile",
    "render_heightmaps": ".tactile",
    "SensorObserver": ".observer",
    "pose_delta": ".observer",
    "normals_from": ".optical",
    "shade": ".optical",
    "lut_from_polytable": ".optical",
    "add_shadows": ".optical",
    "shadow_factor": ".optical",
    "contact_center": ".marker",
    "track_load": ".marker",
    "marker_displacements": ".marker",
    "render_markers": ".marker",
    "marker_config": ".marker",
    "observation_digest": ".digest",
}


def __getattr__(name):
    # torch-dependent modules load on first use so `import paper_2411_04776_b200`
    # stays cheap for config-only users.
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(mod, __name__), name)
