"""Time the reference's own CPU functions against the oracle port that
bench.py's CPU arm runs on the GPU box (the reference cannot travel there).

BUILD CONTAINER ONLY (imports the reference from TACSIM_SRC, default
/root/reference/pkg/src).  Single-threaded, the same seeded configs[4] frames
bench.py uses, per frame:

  reference (BASELINE.md §2 plan): tactile.indentation_from -> the sigma
  pyramid via the gaussian_filter call of tactile.py:219 -> optical.normals_from
  -> optical.shade with a calibrated global table (optical.calibrate) -> uint8
  rule (cli.py:134-139) -> marker.contact_center -> marker.marker_displacements
  -> marker.render_markers (r = 3); with --shadows also optical.add_shadows.
  port: oracle.fast.FastOracle.run (binned LUT in place of the global table).

Writes profiles/r02_cpu_ref_vs_port.json: ms/frame of both and their ratio,
which scales bench.py's cpu_baseline (port) to the reference's own speed.

    OMP_NUM_THREADS=1 python tools/ref_vs_port.py [--frames 24] [--shadows]
"""

import argparse
import json
import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SRC = os.environ.get("TACSIM_SRC", "/root/reference/pkg/src")
sys.path.insert(0, SRC)
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402
import torch  # noqa: E402
from scipy import ndimage  # noqa: E402

import tacsim.marker as mk  # noqa: E402
import tacsim.optical as op  # noqa: E402
import tacsim.tactile as tac  # noqa: E402

from oracle.fast import FastOracle  # noqa: E402
from paper_2411_04776_b200 import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=24)
    ap.add_argument("--shadows", action="store_true")
    a = ap.parse_args()
    torch.set_num_threads(1)
    cfg, n, params, shear, twist = synthetic.workload(4, 0)
    if a.shadows:
        import dataclasses

        d = np.asarray(op.default_lighting().directions, dtype=np.float64)
        cfg = dataclasses.replace(cfg, light_dirs=d, shadow_factor=0.6)
    h, w = cfg.sensor.image_size
    ids = np.linspace(0, n - 1, a.frames).round().astype(np.int64)
    depth = synthetic.height_maps(params.subset(ids), h, w, dtype=torch.float64).numpy()
    sh, tw = shear[ids], twist[ids]
    scfg = tac.SensorConfig(image_size=(h, w), sensing_area=(w * cfg.pixel_pitch, h * cfg.pixel_pitch),
                            gelpad_thickness=cfg.sensor.gelpad_thickness, marker_grid=cfg.sensor.marker_grid)
    lighting = op.default_lighting()
    table = op.calibrate(lighting, scfg)
    mp = mk.MarkerParams(lambda_n=cfg.marker_params.lambda_n)
    rest = mk.grid_rest_positions(scfg)

    def reference(k):
        hm = tac.HeightMap(depth[k], cfg.pixel_pitch)
        ind = tac.indentation_from(hm, scfg)
        acc = np.zeros_like(ind.values)
        for sigma, r in cfg.levels:
            acc += ndimage.gaussian_filter(ind.values, sigma=sigma, mode="nearest", truncate=r / sigma)
        sm = tac.IndentationMap(acc / len(cfg.levels), cfg.pixel_pitch)
        rgb = op.shade(op.normals_from(sm), table)
        if a.shadows:
            rgb = op.add_shadows(rgb, hm, lighting)
        img = np.round(np.clip(rgb, 0.0, 1.0) * 255.0).astype(np.uint8)
        load = mk.contact_center(ind)
        if load.in_contact:
            import dataclasses

            load = dataclasses.replace(load, shear=(float(sh[k, 0]), float(sh[k, 1])), twist=float(tw[k]))
        field = mk.marker_displacements(load, rest, mp)
        return mk.render_markers(field, scfg, background=rgb, dot_radius=3), img

    fast = FastOracle(cfg)
    reference(0)
    fast.run(depth[0], sh[0], tw[0])
    t0 = time.perf_counter()
    for k in range(a.frames):
        reference(k)
    t_ref = (time.perf_counter() - t0) / a.frames
    t0 = time.perf_counter()
    for k in range(a.frames):
        fast.run(depth[k], sh[k], tw[k])
    t_port = (time.perf_counter() - t0) / a.frames
    out = {
        "frames": a.frames, "workload": "configs[4]" + (" + shadows" if a.shadows else ""),
        "threads": 1, "reference_ms_per_frame": 1e3 * t_ref, "port_ms_per_frame": 1e3 * t_port,
        "reference_over_port_time": t_ref / t_port,
        "note": "build container CPU, single thread; bench.py cpu_baseline times the port on the GPU host",
    }
    print(json.dumps(out))
    path = os.path.join(ROOT, "profiles", "r02_cpu_ref_vs_port.json")
    doc = json.load(open(path)) if os.path.exists(path) else {}
    doc[out["workload"]] = out
    json.dump(doc, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
