"""Pin the CPU oracle to golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import marker, optical, tactile


class TestTactileGolden:
    def test_indentation(self, golden):
        g = golden("tactile")
        ind = tactile.indentation_from(g["depth"], float(g["rest"]))
        assert np.array_equal(ind, g["ind"])

    @pytest.mark.parametrize("ki", range(5))
    def test_kernel_size_pyramid(self, golden, ki):
        g = golden("tactile")
        levels = tactile.levels_from_kernel_sizes(g[f"ksizes_{ki}"])
        out = tactile.smooth_pyramid(g["ind"], levels)
        ref = g[f"smooth_k{ki}"]
        assert np.abs(out - ref).max() <= 1e-15 * max(1.0, np.abs(ref).max()) + 1e-20

    @pytest.mark.parametrize("si", range(3))
    def test_sigma_pyramid(self, golden, si):
        g = golden("tactile")
        levels = tactile.levels_from_sigmas(g[f"sigmas_{si}"])
        out = tactile.smooth_pyramid(g["ind"], levels)
        ref = g[f"smooth_s{si}"]
        assert np.abs(out - ref).max() <= 1e-15 * max(1.0, np.abs(ref).max()) + 1e-20

    def test_identity_level_exact(self, golden):
        g = golden("tactile")
        out = tactile.smooth_pyramid(g["ind"], tactile.levels_from_kernel_sizes([1]))
        assert np.array_equal(out, g["smooth_k2"])

    def test_kernel_validation(self):
        for bad in ([4], [11, 5], []):
            with pytest.raises(ValueError):
                tactile.levels_from_kernel_sizes(bad)


class TestOpticalGolden:
    def test_gradient_known_answer(self, golden):
        g = golden("optical")
        gy, gx = optical.gradient(np.array([[0.0, 1.0, 4.0, 9.0]] * 2), 0.5)
        assert np.array_equal(gx[0], g["gradient_known"])

    def test_normals(self, golden):
        g = golden("optical")
        n = optical.normals_from(g["smooth"], 2.66e-5)
        assert np.abs(n - g["normals"]).max() < 1e-12

    def test_tilted_plane(self, golden):
        g = golden("optical")
        n = optical.normals_from(g["tilted"], 2.5e-5)
        assert np.abs(n - g["tilted_normals"]).max() < 1e-12

    def test_global_shade(self, golden):
        g = golden("optical")
        out, _ = optical.shade_global(g["normals"], g["coeffs"], g["background"])
        assert np.abs(out - g["shaded"]).max() < 1e-12
        assert np.array_equal(optical.quantize_u8(out), g["shaded_u8"])

    def test_single_bin_lut_matches_reference_shade(self, golden):
        """The binned LUT's only reference anchor: every bin = global table."""
        g = golden("optical")
        lut = optical.lut_from_global(g["coeffs"], 125, 180)
        rgb, _ = optical.shade_lut(g["smooth"], 2.66e-5, lut, g["background"] * 255.0, 1.0)
        d = np.abs(rgb.astype(int) - g["shaded_u8"].astype(int))
        assert d.max() <= 1
        assert (d == 0).mean() >= 0.999


class TestMarkerGolden:
    def test_contact_center(self, golden):
        g = golden("marker")
        for v, ref in zip(g["cc_maps"], g["cc"]):
            c = marker.contact_center(v, 2.66e-5)
            got = [c["cx"], c["cy"], c["dmax"], float(c["in_contact"])]
            assert np.allclose(got, ref, rtol=1e-12, atol=1e-20)

    def test_two_pixel(self, golden):
        g = golden("marker")
        two = np.zeros((9, 9))
        two[4, 2] = 1e-4
        two[4, 6] = 3e-4
        c = marker.contact_center(two, 2.66e-5)
        assert np.allclose([c["cx"], c["cy"], c["dmax"], 1.0], g["cc_two"], rtol=1e-12, atol=1e-20)

    def test_grid(self, golden):
        g = golden("marker")
        grid = marker.grid_rest_positions(7, 9, 64 * 2.66e-5, 48 * 2.66e-5)
        assert np.array_equal(grid, g["grid"])

    def test_displacements(self, golden):
        g = golden("marker")
        for ld, ref in zip(g["loads"], g["disps"]):
            load = dict(cx=ld[0], cy=ld[1], dmax=ld[2], sx=ld[3], sy=ld[4], twist=ld[5],
                        in_contact=bool(ld[6]))
            u = marker.marker_displacements(load, g["grid"])
            assert np.abs(u - ref).max() <= 1e-15 * max(1e-9, np.abs(ref).max())

    def test_lambda_n(self, golden):
        g = golden("marker")
        load = dict(cx=1e-4, cy=-2e-4, dmax=9e-4, sx=1e-4, sy=2e-4, twist=0.05, in_contact=True)
        p = (0.3, 0.8e-3, 5e-3, 0.5, 4e-3)
        u = marker.marker_displacements(load, g["grid"], p)
        assert np.abs(u - g["disp_lambda_n_08"]).max() < 1e-18

    def test_track_load(self, golden):
        g = golden("marker")
        state = dict(cx=0.0, cy=0.0, dmax=0.0, sx=0.0, sy=0.0, twist=0.0, in_contact=False)
        for inp, ref in zip(g["track_in"], g["track_out"]):
            contact = dict(cx=inp[3], cy=inp[4], dmax=inp[5], in_contact=bool(inp[6]))
            state = marker.track_load(state, inp[:3], contact)
            got = [state["cx"], state["cy"], state["dmax"], state["sx"], state["sy"],
                   state["twist"], float(state["in_contact"])]
            assert np.allclose(got, ref, rtol=1e-12, atol=1e-18)

    def test_circle_stencil(self, golden):
        g = golden("marker")
        yy, xx = np.mgrid[0:64, 0:64]
        for r, ref in enumerate(g["circle_stencils"]):
            assert np.array_equal((yy - 32) ** 2 + (xx - 32) ** 2 <= r * r, ref)

    def test_render(self, golden):
        g = golden("marker")
        o = golden("optical")
        pos = g["grid"] + g["render_disp"]
        bg = optical.quantize_u8(o["shaded"][0])
        img = marker.render_markers(bg, pos, 2.66e-5, 3)
        assert np.array_equal(img, g["render_r3"])
        grey = np.full((48, 64, 3), 230, np.uint8)
        img4 = marker.render_markers(grey, pos, 2.66e-5, 4)
        assert np.array_equal(img4, g["render_r4_grey"])


class TestShadowsGolden:
    """add_shadows (optical.py:261-300) restated: per-light march, soft edge,
    multiplicative factor; pinned on the reference's own outputs."""

    def test_default_and_grazing_lights(self, golden):
        g = golden("shadows")
        for mi, hm in enumerate(g["maps"]):
            out = optical.add_shadows(g["rgb"], -hm, 2.66e-5, g["dirs_default"])
            assert np.abs(out - g[f"default_{mi}"]).max() < 1e-12
            out = optical.add_shadows(g["rgb"], -hm, 2.66e-5, g["dirs_graze"], factor=0.3,
                                      max_steps=40, softness=2e-5)
            assert np.abs(out - g[f"graze_{mi}"]).max() < 1e-12

    def test_factor_form_matches(self, golden):
        g = golden("shadows")
        hm = g["maps"][1]
        f = optical.shadow_factor(-hm, 2.66e-5, g["dirs_default"])
        assert np.abs(g["rgb"] * f[..., None] - g["default_1"]).max() < 1e-12
        assert (f < 1).any() and (f == 1).any()

    def test_flat_map_identity(self, golden):
        g = golden("shadows")
        assert np.array_equal(g["default_2"], g["rgb"])


class TestRasterGolden:
    """Row f2: oracle render_heightmap vs the reference's own depth maps
    (tests/golden/raster.npz, REF/tactile.py:129-190), bit for bit."""

    def test_cases_bit_exact(self, golden):
        g = golden("raster")
        for k in range(int(g["n_cases"])):
            d = tactile.render_heightmap(g[f"verts_cam_{k}"], g[f"tris_{k}"], 48, 64, 2.66e-5, 4e-3)
            assert np.array_equal(d, g[f"depth_{k}"]), k

    def test_empty_scene_is_rest(self):
        d = tactile.render_heightmap(np.zeros((0, 3)), np.zeros((0, 3), np.int64), 8, 10, 1e-4, 4e-3)
        assert np.array_equal(d, np.full((8, 10), 4e-3))

    def test_triangle_order_invariance(self, golden):
        g = golden("raster")
        t = g["tris_0"]
        perm = np.random.default_rng(3).permutation(len(t))
        a = tactile.render_heightmap(g["verts_cam_0"], t, 48, 64, 2.66e-5, 4e-3)
        b = tactile.render_heightmap(g["verts_cam_0"], t[perm], 48, 64, 2.66e-5, 4e-3)
        assert np.array_equal(a, b)

    def test_camera_frame_matrix_matches_pose_inverse(self):
        from paper_2411_04776_b200.tactile import _camera_frame

        rng = np.random.default_rng(5)
        c, s = np.cos(0.3), np.sin(0.3)
        m = np.eye(4)
        m[:3, :3] = [[c, -s, 0], [s, c, 0], [0, 0, 1]]
        m[:3, 3] = [0.1, -0.2, 0.3]
        p = rng.normal(size=(20, 3))
        back = _camera_frame(p @ m[:3, :3].T + m[:3, 3], m)
        assert np.allclose(back, p, atol=1e-14)
