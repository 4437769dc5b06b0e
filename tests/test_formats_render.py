"""Row f4: reference file formats (CPU) and the `render` replay against the
reference's own `tacsim calibrate` + `tacsim render` outputs (GPU)."""

import os

import numpy as np
import pytest

from paper_2411_04776_b200 import formats


def _write_case(tmp_path, g):
    files = []
    for i in range(4):
        f = tmp_path / f"m{i}.raw"
        f.write_bytes(g[f"raw_{i}"].tobytes())
        files.append(str(f))
    (tmp_path / "table.json").write_bytes(g["table_json"].tobytes())
    (tmp_path / "table.png").write_bytes(g["table_png"].tobytes())
    return files


class TestFormats:
    def test_raw_maps_byte_identical_to_reference(self, golden, tmp_path):
        g = golden("render")
        for i in range(4):
            ref = g[f"raw_{i}"].tobytes()
            src = tmp_path / "ref.raw"
            src.write_bytes(ref)
            v, pitch = formats.load_map_raw(str(src))
            out = tmp_path / "ours.raw"
            formats.save_map_raw(str(out), v, pitch)
            assert out.read_bytes() == ref

    def test_raw_errors(self, tmp_path):
        p = tmp_path / "bad.raw"
        p.write_bytes(b"XXXX" + bytes(12))
        with pytest.raises(formats.MeshFormatError):
            formats.load_map_raw(str(p))
        formats.save_map_raw(str(p), np.zeros((4, 5)), 1e-5)
        p.write_bytes(p.read_bytes()[:-4])
        with pytest.raises(formats.MeshFormatError):
            formats.load_map_raw(str(p))

    def test_markers_csv_round_trip(self, tmp_path):
        rng = np.random.default_rng(3)
        rest, disp = rng.normal(size=(3, 4, 2)), rng.normal(size=(3, 4, 2)) * 1e-4
        p = str(tmp_path / "m.csv")
        formats.save_markers_csv(p, rest, disp)
        r2, d2 = formats.load_markers_csv(p)
        assert np.array_equal(r2, rest) and np.array_equal(d2, disp)

    def test_polytable_loads(self, golden, tmp_path):
        pytest.importorskip("cv2")
        g = golden("render")
        _write_case(tmp_path, g)
        coeffs, bg = formats.load_polytable(str(tmp_path / "table.json"), str(tmp_path / "table.png"))
        assert coeffs.shape == (3, 6) and bg.shape == (480, 640, 3)


@pytest.mark.gpu
class TestRenderReplay:
    def test_matches_reference_cli(self, golden, tmp_path, capsys):
        from paper_2411_04776_b200 import render

        g = golden("render")
        files = _write_case(tmp_path, g)
        out = tmp_path / "out"
        code = render.main(files + ["--table", str(tmp_path / "table.json"), "--table-png",
                                    str(tmp_path / "table.png"), "--out", str(out)])
        assert code == 0
        lines = [l for l in capsys.readouterr().out.strip().split("\n") if "contact pixels" in l]
        counts = [int(l.rsplit(" ", 1)[1]) for l in lines]
        assert counts == g["counts"].tolist()
        for i in range(4):
            got = formats.read_rgb_png(str(out / f"m{i}_tactile.png")).astype(int)
            d = np.abs(got - g[f"png_{i}"].astype(int))
            assert d.max() <= 1 or (d > 1).mean() <= 1e-3, (i, d.max(), (d > 1).mean())
            assert (d <= 1).mean() >= 0.999
            rest, disp = formats.load_markers_csv(str(out / f"m{i}_markers.csv"))
            assert np.array_equal(rest, g[f"rest_{i}"])
            ref = g[f"disp_{i}"]
            den = max(np.abs(ref).max(), 1e-30)
            assert np.abs(disp - ref).max() <= 1e-4 * den

    def test_missing_table_is_config_error(self, tmp_path):
        from paper_2411_04776_b200 import render

        p = tmp_path / "flat.raw"
        formats.save_map_raw(str(p), np.full((8, 8), 4e-3), 2.5e-5)
        assert render.main([str(p), "--out", str(tmp_path / "r")]) == render.EXIT_CONFIG
        assert render.main([str(p), "--table", "no.json", "--table-png", "no.png"]) == render.EXIT_CONFIG
