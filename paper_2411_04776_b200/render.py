"""``render``: offline replay of recorded height maps on the GPU.

Mirror of ``tacsim render`` (REF/cli.py:274-301): for every TAC1 raw height
map, indentation_from -> smooth_pyramid(DEFAULT_PYRAMID) -> normals -> shade
with the calibrated table -> add_shadows(default lighting, factor 0.6) ->
``<stem>_tactile.png``; contact_center -> marker_displacements ->
``<stem>_markers.csv``; prints the contact-pixel count (indentation > 1e-5).
Same exit codes (0 ok, 2 config, 4 I/O).  The maps are batched through one
fused launch per batch plus the shadow march.

    python -m paper_2411_04776_b200.render maps/*.raw --table t.json --table-png t.png --out out/
"""

import argparse
import os
import sys

import numpy as np

EXIT_OK, EXIT_CONFIG, EXIT_SOLVER, EXIT_IO = 0, 2, 3, 4


def _default_light_dirs():
    """tacsim default_lighting() (REF/optical.py:68-79), normalised as
    LightingModel does (REF/optical.py:36-45)."""
    el = np.deg2rad(35.0)
    az = np.deg2rad([0.0, 120.0, 240.0])
    d = np.stack([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.full(3, np.sin(el))], axis=1)
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def render_files(files, table, table_png, out, batch=256, device="cuda"):
    import torch

    from . import TactilePipeline
    from .config import (DEFAULT_PYRAMID, PipelineConfig, SensorConfig, grid_rest_positions,
                         levels_from_kernel_sizes)
    from .errors import InvalidArgumentError
    from .formats import load_map_raw, load_polytable, save_markers_csv, write_rgb_png
    from .marker import contact_center, marker_config
    from .optical import lut_from_polytable

    coeffs, background = load_polytable(table, table_png)
    sensor = SensorConfig()  # the ball_rolling scene's sensor (REF/envs.py:164-189)
    maps = [load_map_raw(f) for f in files]
    h, w = maps[0][0].shape
    pitch = maps[0][1]
    for v, p in maps:
        if v.shape != (h, w) or p != pitch:
            raise InvalidArgumentError("all maps of one render call must share shape and pitch")
    if background.shape[:2] != (h, w):
        raise InvalidArgumentError("normals and background shapes differ")
    map_sensor = SensorConfig((h, w), (w * pitch, h * pitch), sensor.gelpad_thickness, sensor.marker_grid)
    grid = grid_rest_positions(sensor)
    cfg = PipelineConfig(
        sensor=map_sensor,
        levels=levels_from_kernel_sizes(DEFAULT_PYRAMID),
        lut=lut_from_polytable(coeffs, 1, 1),
        background=(background * 255.0).astype(np.float32),
        rest_grid=grid,
        light_dirs=_default_light_dirs(),
        shadow_factor=0.6,
        shadow_steps=80,
        shadow_softness=5e-5,
    )
    count_cfg = marker_config(map_sensor, threshold=1e-5, rest_grid=grid)
    pipe = TactilePipeline(cfg, device)
    os.makedirs(out, exist_ok=True)
    counts = []
    for s in range(0, len(files), batch):
        chunk = files[s:s + batch]
        depth = torch.as_tensor(np.stack([maps[s + k][0] for k in range(len(chunk))])).to(device)
        n = depth.shape[0]
        zeros2 = torch.zeros((n, 2), dtype=torch.float64, device=device)
        zeros1 = torch.zeros((n,), dtype=torch.float64, device=device)
        obs = pipe.simulate(depth, zeros2, zeros1, splat=False)
        _, summ = contact_center(depth, count_cfg, input_kind="depth")
        rgb = obs.rgb.cpu().numpy()
        disp = obs.disp.cpu().numpy().astype(np.float64)
        npix = np.rint(summ[:, 1].cpu().numpy().astype(np.float64) / (pitch * pitch)).astype(np.int64)
        for k, path in enumerate(chunk):
            stem = os.path.splitext(os.path.basename(path))[0]
            write_rgb_png(os.path.join(out, f"{stem}_tactile.png"), rgb[k])
            save_markers_csv(os.path.join(out, f"{stem}_markers.csv"), grid, disp[k])
            print(f"{path}: contact pixels {int(npix[k])}")
            counts.append(int(npix[k]))
    return counts


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="render", description="turn recorded height maps into tactile frames")
    ap.add_argument("files", nargs="+", help="height map .raw files")
    ap.add_argument("--table", help="calibrated table JSON")
    ap.add_argument("--table-png", help="calibrated table background PNG")
    ap.add_argument("--out", default="render", help="output directory")
    ap.add_argument("--batch", type=int, default=256, help="maps per GPU launch")
    args = ap.parse_args(argv)
    from .errors import InvalidArgumentError, TacsimError
    from .formats import MeshFormatError

    if not args.table or not args.table_png:
        print("error: rendering needs a calibrated table: pass --table/--table-png", file=sys.stderr)
        return EXIT_CONFIG
    for p in (args.table, args.table_png):
        if not os.path.exists(p):
            print(f"error: missing table file {p}: run calibrate first", file=sys.stderr)
            return EXIT_CONFIG
    try:
        render_files(args.files, args.table, args.table_png, args.out, args.batch)
    except InvalidArgumentError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except (MeshFormatError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_IO
    except TacsimError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_SOLVER
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
