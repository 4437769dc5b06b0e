"""Generate the golden vectors that pin the oracle to the reference.

Runs ONLY in the build container, where the reference package is importable
(``TACSIM_SRC``, default ``/root/reference/pkg/src``).  It calls the
reference's own public functions (tactile / optical / marker, plus the
``scipy.ndimage.gaussian_filter`` call of tactile.py:219 for the sigma-keyed
pyramid and ``cv2.circle`` for the dot stencil) on small seeded inputs and
writes ``tests/golden/{tactile,optical,marker}.npz``.  The fixtures are
committed; the GPU box never needs the reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
"""

import os
import sys

import numpy as np

SRC = os.environ.get("TACSIM_SRC", "/root/reference/pkg/src")
sys.path.insert(0, SRC)
sys.dont_write_bytecode = True

import cv2  # noqa: E402
from scipy import ndimage  # noqa: E402

import tacsim.geometry as geo  # noqa: E402
import tacsim.marker as mk  # noqa: E402
import tacsim.optical as op  # noqa: E402
import tacsim.tactile as tac  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
H, W = 48, 64
PITCH = 2.66e-5
REST = 4e-3
CFG = tac.SensorConfig(
    image_size=(H, W), sensing_area=(W * PITCH, H * PITCH), gelpad_thickness=REST,
    marker_grid=(7, 9),
)


def sphere_depth(h, w, pitch, radius, pen, cx=0.0, cy=0.0):
    ys = (np.arange(h) + 0.5 - 0.5 * h) * pitch - cy
    xs = (np.arange(w) + 0.5 - 0.5 * w) * pitch - cx
    gx, gy = np.meshgrid(xs, ys)
    cap = np.sqrt(np.clip(radius * radius - gx * gx - gy * gy, 0.0, None))
    ind = np.clip(pen - radius + cap, 0.0, None)
    return REST - ind


def tactile_cases():
    rng = np.random.default_rng(1234)
    depths = np.stack(
        [
            sphere_depth(H, W, PITCH, 1e-3, 2e-4, 3 * PITCH, -2 * PITCH),
            # exercises both clamps: beyond the rest surface and behind the camera plane
            rng.uniform(-5e-4, REST + 5e-4, size=(H, W)),
            np.full((H, W), REST),
        ]
    )
    sigma_sets = [(1.0, 2.0, 4.0), (1.0, 2.0, 4.0, 8.0), (0.5, 1.5)]
    kernel_sets = [(5, 11, 21, 31), (3,), (1,), (1, 5), (3, 7, 9)]
    out = dict(depth=depths, pitch=PITCH, rest=REST)
    inds = []
    for d in depths:
        inds.append(tac.indentation_from(tac.HeightMap(d, PITCH), CFG).values)
    out["ind"] = np.stack(inds)
    for ki, ks in enumerate(kernel_sets):
        out[f"ksizes_{ki}"] = np.array(ks)
        out[f"smooth_k{ki}"] = np.stack(
            [tac.smooth_pyramid(tac.IndentationMap(v, PITCH), ks).values for v in inds]
        )
    for si, ss in enumerate(sigma_sets):
        out[f"sigmas_{si}"] = np.array(ss)
        res = []
        for v in inds:
            acc = np.zeros_like(v)
            for s in ss:
                r = int(np.ceil(3 * s - 1e-12))
                # the same call as tactile.py:219-221 with sigma supplied directly
                acc += ndimage.gaussian_filter(v, sigma=s, mode="nearest", truncate=r / s)
            res.append(acc / len(ss))
        out[f"smooth_s{si}"] = np.stack(res)
    return out


def optical_cases(tact):
    table = op.calibrate(op.default_lighting(), CFG)
    smooth = tact["smooth_k0"]
    normals = np.stack([op.normals_from(tac.IndentationMap(v, PITCH)) for v in smooth])
    shaded = np.stack([op.shade(n, table) for n in normals])
    # analytic known answers (test_optical.py:65-85)
    theta = 0.2
    xs = (np.arange(60) + 0.5) * 2.5e-5
    tilted = np.tile(xs * np.tan(theta), (40, 1))
    return dict(
        smooth=smooth,
        normals=normals,
        coeffs=table.coeffs,
        background=table.background,
        shaded=shaded,
        shaded_u8=np.round(np.clip(shaded, 0.0, 1.0) * 255.0).astype(np.uint8),
        tilted=tilted,
        tilted_normals=op.normals_from(tilted, 2.5e-5),
        gradient_known=np.gradient(np.array([0.0, 1.0, 4.0, 9.0]), 0.5),
    )


def shadow_cases(tact, opt):
    """add_shadows (optical.py:261-300) on the press maps, default lighting and
    a single grazing light, factor 0.6 and 0.3."""
    lights = op.default_lighting()
    graze = op.LightingModel(np.array([[0.94, 0.0, 0.34]] * 3), np.eye(3), np.zeros(3))
    bumpy = np.full((H, W), REST)
    bumpy[20:26, 30:36] = REST - 1e-3
    maps = np.stack([tact["depth"][0], bumpy, tact["depth"][2]])
    rgb = opt["shaded"][0]
    out = dict(maps=maps, rgb=rgb, dirs_default=lights.directions, dirs_graze=graze.directions)
    for mi, hmv in enumerate(maps):
        hm = tac.HeightMap(hmv, PITCH)
        out[f"default_{mi}"] = op.add_shadows(rgb, hm, lights)
        out[f"graze_{mi}"] = op.add_shadows(rgb, hm, graze, factor=0.3, max_steps=40, softness=2e-5)
    return out


def marker_cases(tact, opt):
    rng = np.random.default_rng(99)
    grid = mk.grid_rest_positions(CFG)
    out = dict(grid=grid)
    # contact_center on each indentation + hand cases (test_marker.py:54-99)
    two = np.zeros((9, 9))
    two[4, 2] = 1e-4
    two[4, 6] = 3e-4
    maps = list(tact["ind"]) + [np.full((H, W), 4e-5)]
    cc = []
    for v in maps:
        s = mk.contact_center(tac.IndentationMap(v, PITCH))
        cc.append([*s.contact_center, s.max_indentation, float(s.in_contact)])
    out["cc_maps"] = np.stack(maps)
    out["cc"] = np.array(cc)
    s = mk.contact_center(tac.IndentationMap(two, PITCH))
    out["cc_two"] = np.array([*s.contact_center, s.max_indentation, float(s.in_contact)])
    # displacements for a spread of loads
    loads = []
    disps = []
    for i in range(12):
        in_contact = i % 4 != 3
        if in_contact:
            c = rng.uniform(-1e-3, 1e-3, 2) if i != 5 else grid[3, 4]
            ld = mk.LoadState(tuple(c), float(rng.uniform(0, 1.2e-3)),
                              tuple(rng.uniform(-3e-4, 3e-4, 2)),
                              float(rng.uniform(-0.0873, 0.0873)), True)
        else:
            ld = mk.LoadState.zero()
        loads.append([*ld.contact_center, ld.max_indentation, *ld.shear, ld.twist, float(ld.in_contact)])
        disps.append(mk.marker_displacements(ld, grid).displacements)
    out["loads"] = np.array(loads)
    out["disps"] = np.stack(disps)
    lam = mk.MarkerParams(lambda_n=0.8e-3)
    out["disp_lambda_n_08"] = mk.marker_displacements(
        mk.LoadState((1e-4, -2e-4), 9e-4, (1e-4, 2e-4), 0.05, True), grid, lam
    ).displacements
    # track_load over a scripted contact sequence (marker.py:124-140)
    state = mk.LoadState.zero()
    seq_in, seq_out = [], []
    for t in range(10):
        contact_on = t not in (0, 6)
        dx, dy, rz = rng.uniform(-1e-4, 1e-4), rng.uniform(-1e-4, 1e-4), rng.uniform(-0.02, 0.02)
        delta = geo.Pose.from_rotvec([dx, dy, 0.0], [0.0, 0.0, rz])
        contact = mk.LoadState((1e-4 * t, -5e-5 * t), 1e-4 * (t + 1), (0, 0), 0.0, True) if contact_on else mk.LoadState.zero()
        state = mk.track_load(state, delta, contact)
        seq_in.append([dx, dy, float(delta.rot().as_rotvec()[2]), *contact.contact_center,
                       contact.max_indentation, float(contact.in_contact)])
        seq_out.append([*state.contact_center, state.max_indentation, *state.shear,
                        state.twist, float(state.in_contact)])
    out["track_in"] = np.array(seq_in)
    out["track_out"] = np.array(seq_out)
    # dot rendering: shaded background (r=3) and default 230 grey (r=4),
    # with displacements that push dots across the borders and onto .5 ties
    disp = rng.uniform(-8 * PITCH, 8 * PITCH, size=grid.shape)
    disp[0, 0] = (-30 * PITCH, -30 * PITCH)  # fully outside
    disp[6, 8] = (4 * PITCH, 3 * PITCH)  # clipped at bottom-right
    disp[3, 3] = (0.0, 0.0)
    field = mk.MarkerField(grid, disp)
    bg = opt["shaded"][0]
    out["render_disp"] = disp
    out["render_r3"] = mk.render_markers(field, CFG, background=bg, dot_radius=3)
    out["render_r4_grey"] = mk.render_markers(field, CFG, dot_radius=4)
    # cv2 filled-circle stencil == {dx^2+dy^2 <= r^2}
    sten = []
    for r in range(0, 13):
        img = np.zeros((64, 64), np.uint8)
        cv2.circle(img, (32, 32), r, 255, -1)
        sten.append(img > 0)
    out["circle_stencils"] = np.stack(sten)
    return out


def render_cases():
    """`tacsim calibrate` + `tacsim render` (REF/cli.py:274-319) run end to end
    on four 480x640 TAC1 maps: flat, sphere presses of 0.4 and 0.8 mm (as
    REF/tests/test_cli.py:148-161) and an off-centre cylinder."""
    import contextlib
    import io
    import tempfile

    import tacsim.cli as cli

    cfg = tac.SensorConfig()
    h, w = cfg.image_size
    p, th = cfg.pixel_pitch, cfg.gelpad_thickness
    yy, xx = np.mgrid[0:h, 0:w]
    x = (xx + 0.5 - 0.5 * w) * p
    y = (yy + 0.5 - 0.5 * h) * p

    def press(depth, r=5e-3, cx=0.0, cy=0.0):
        rho2 = (x - cx) ** 2 + (y - cy) ** 2
        sph = th - depth + r - np.sqrt(np.maximum(0.0, r * r - rho2))
        return np.where(rho2 <= r * r, np.minimum(np.full((h, w), th), sph), th)

    perp = (x - 1e-3) * np.sin(0.4) - (y + 5e-4) * np.cos(0.4)
    cyl = np.where(np.abs(perp) < 3e-3, th - np.maximum(0.0, 6e-4 - 3e-3 + np.sqrt(np.maximum(0, 9e-6 - perp * perp))), th)
    maps = [np.full((h, w), th), press(4e-4), press(8e-4, cx=2e-3, cy=-1e-3), np.minimum(cyl, th)]
    out = {}
    with tempfile.TemporaryDirectory() as d:
        files = []
        for i, m in enumerate(maps):
            f = os.path.join(d, f"m{i}.raw")
            tac.save_heightmap_raw(f, tac.HeightMap(m, p))
            files.append(f)
            out[f"raw_{i}"] = np.frombuffer(open(f, "rb").read(), dtype=np.uint8)
        cal = os.path.join(d, "cal")
        with contextlib.redirect_stdout(io.StringIO()):
            assert cli.main(["calibrate", "--out", cal]) == 0
        buf = io.StringIO()
        rd = os.path.join(d, "r")
        with contextlib.redirect_stdout(buf):
            assert cli.main(["render", *files, "--table", os.path.join(cal, "table.json"),
                             "--table-png", os.path.join(cal, "table.png"), "--out", rd]) == 0
        out["table_json"] = np.frombuffer(open(os.path.join(cal, "table.json"), "rb").read(), dtype=np.uint8)
        out["table_png"] = np.frombuffer(open(os.path.join(cal, "table.png"), "rb").read(), dtype=np.uint8)
        out["counts"] = np.array([int(l.rsplit(" ", 1)[1]) for l in buf.getvalue().strip().split("\n")])
        for i in range(len(maps)):
            out[f"png_{i}"] = cv2.imread(os.path.join(rd, f"m{i}_tactile.png"))[:, :, ::-1]
            field = mk.load_markers_csv(os.path.join(rd, f"m{i}_markers.csv"))
            out[f"disp_{i}"] = field.displacements
            out[f"rest_{i}"] = field.rest_positions
    return out


def raster_cases():
    """render_heightmap (tactile.py:129-190) on meshes at several poses: the
    camera-frame vertices the reference rasterises and its depth maps."""
    out = {}
    ident = geo.Pose()
    cases = []
    sph = geo.icosphere_surface(1.2e-3, 3)
    cases.append((sph.vertices + np.array([0.0, 0.0, REST - 4e-4 + 1.2e-3]), sph.triangles, ident))
    cases.append((sph.vertices + np.array([3.1e-4, -2.2e-4, REST - 7e-4 + 1.2e-3]), sph.triangles, ident))
    world = geo.Pose.from_rotvec([0.03, -0.02, 0.05], [0.4, -0.3, 0.9])
    cases.append((world.apply(sph.vertices + np.array([1e-4, 0.0, REST - 5e-4 + 1.2e-3])), sph.triangles, world))
    plate_v = np.array([[-1.0, -1.0, REST - 2e-4], [1.0, -1.0, REST - 2e-4], [1.0, 1.0, REST - 1e-4],
                        [-1.0, 1.0, REST - 1e-4]]) * np.array([1e-3, 1e-3, 1.0])
    cases.append((plate_v, np.array([[0, 1, 2], [0, 2, 3]]), ident))
    cases.append((plate_v + np.array([0.0, 0.0, 5e-4]), np.array([[0, 1, 2], [0, 2, 3]]), ident))  # beyond rest
    small = geo.icosphere_surface(2e-4, 2)
    cases.append((small.vertices + np.array([-7e-4, 5e-4, REST - 1e-4 + 2e-4]), small.triangles, ident))
    for k, (vw, tri, pose) in enumerate(cases):
        hm = tac.render_heightmap([(vw, tri)], pose, CFG)
        out[f"verts_cam_{k}"] = pose.inverse().apply(vw)
        out[f"tris_{k}"] = np.asarray(tri, dtype=np.int32)
        out[f"depth_{k}"] = hm.values
    out["n_cases"] = np.array(len(cases))
    return out


def main():
    tact = tactile_cases()
    opt = optical_cases(tact)
    mark = marker_cases(tact, opt)
    shad = shadow_cases(tact, opt)
    np.savez_compressed(os.path.join(OUT, "shadows.npz"), **shad)
    np.savez_compressed(os.path.join(OUT, "render.npz"), **render_cases())
    np.savez_compressed(os.path.join(OUT, "raster.npz"), **raster_cases())
    np.savez_compressed(os.path.join(OUT, "tactile.npz"), **tact)
    np.savez_compressed(os.path.join(OUT, "optical.npz"), **opt)
    np.savez_compressed(os.path.join(OUT, "marker.npz"), **mark)
    for name in ("tactile", "optical", "marker", "shadows", "render"):
        p = os.path.join(OUT, f"{name}.npz")
        print(p, os.path.getsize(p))


if __name__ == "__main__":
    main()
