"""CPU-side checks of the C-ABI library and the host logic (no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2411_04776_b200 import _lib
from paper_2411_04776_b200.config import (
    MarkerParams,
    PipelineConfig,
    SensorConfig,
    levels_from_kernel_sizes,
    levels_from_sigmas,
)
from paper_2411_04776_b200.errors import InvalidArgumentError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tac_b200.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tac_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    syms = header_symbols()
    for name in ("tac_ctx_create", "tac_pipeline", "tac_contact_blur", "tac_shade", "tac_contact",
                 "tac_track_load", "tac_marker_displacements", "tac_render_markers", "tac_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert set(header_symbols()) == set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def _cfg(**over):
    c = _lib.TacConfig()
    c.height, c.width = 16, 24
    c.pixel_pitch = 2.66e-5
    c.gel_thickness = 4e-3
    c.n_levels = 3
    for i, (s, r) in enumerate(levels_from_sigmas((1, 2, 4))):
        c.sigma[i], c.radius[i] = s, r
    c.mag_bins, c.dir_bins = 2, 3
    c.g_max = 1.0
    lut = np.zeros((2, 3, 3, 6), np.float32)
    bg = np.full((16, 24, 3), 100.0, np.float32)
    c.lut = lut.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    c.background = bg.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    c.marker_rows, c.marker_cols = 3, 4
    c.k_n, c.lambda_n, c.lambda_s, c.k_t, c.lambda_t = 0.3, 4e-3, 5e-3, 0.5, 4e-3
    c.contact_threshold = 5e-5
    c.dot_radius = 3
    for k, v in over.items():
        if k == "radius":
            c.radius[0] = v
        else:
            setattr(c, k, v)
    return c, (lut, bg)


@pytest.mark.parametrize(
    "field,value,status",
    [
        ("height", 1, _lib.TAC_ERR_INVALID),
        ("pixel_pitch", 0.0, _lib.TAC_ERR_INVALID),
        ("gel_thickness", -1.0, _lib.TAC_ERR_INVALID),
        ("n_levels", 0, _lib.TAC_ERR_INVALID),
        ("n_levels", 9, _lib.TAC_ERR_INVALID),
        ("radius", 25, _lib.TAC_ERR_UNSUPPORTED),
        ("radius", -1, _lib.TAC_ERR_INVALID),
        ("g_max", 0.0, _lib.TAC_ERR_INVALID),
        ("lambda_s", 0.0, _lib.TAC_ERR_INVALID),
        ("k_n", float("nan"), _lib.TAC_ERR_INVALID),
        ("contact_threshold", 0.0, _lib.TAC_ERR_INVALID),
        ("dot_radius", 99, _lib.TAC_ERR_UNSUPPORTED),
    ],
)
def test_ctx_create_validates_before_touching_cuda(field, value, status):
    lib = _lib.load()
    c, keep = _cfg(**{field: value})
    h = ctypes.c_void_p()
    assert lib.tac_ctx_create(ctypes.byref(c), ctypes.byref(h)) == status
    assert lib.tac_last_error()
    with pytest.raises(InvalidArgumentError):
        _lib.check(status)


def test_nonfinite_table_rejected():
    lib = _lib.load()
    c, (lut, bg) = _cfg()
    bg[3, 4, 1] = np.nan
    h = ctypes.c_void_p()
    assert lib.tac_ctx_create(ctypes.byref(c), ctypes.byref(h)) == _lib.TAC_ERR_INVALID
    assert b"finite" in lib.tac_last_error()


def test_null_context_calls_fail_cleanly():
    lib = _lib.load()
    assert lib.tac_pipeline(None, None, None) == _lib.TAC_ERR_INVALID
    assert lib.tac_shade(None, None, None, 0, None) == _lib.TAC_ERR_INVALID
    assert lib.tac_shade_ex(None, None, None, None, 0, None) == _lib.TAC_ERR_INVALID
    assert lib.tac_timing_begin(None, 4) == _lib.TAC_ERR_INVALID
    assert lib.tac_timing_end(None, None, None) == _lib.TAC_ERR_INVALID
    assert lib.tac_render_heightmap(None, None, 0, None, 0, None, 1, None) == _lib.TAC_ERR_INVALID
    assert lib.tac_pipeline_profile(None, None, None, 1, None) == _lib.TAC_ERR_INVALID
    assert lib.tac_pipeline_launches(None, 10) == 0
    assert lib.tac_workspace_bytes(None, 10) == 0


def test_valid_config_without_gpu_is_a_cuda_error():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _lib.load()
    c, keep = _cfg()
    h = ctypes.c_void_p()
    assert lib.tac_ctx_create(ctypes.byref(c), ctypes.byref(h)) == _lib.TAC_ERR_CUDA


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2411_04776_b200 import NativeLibraryError, TactilePipeline
    from paper_2411_04776_b200.synthetic import baseline_config

    cfg, _ = baseline_config(0)
    with pytest.raises(NativeLibraryError):
        TactilePipeline(cfg)


def test_missing_library_fails_loudly(tmp_path):
    from paper_2411_04776_b200.errors import NativeLibraryError

    with pytest.raises(NativeLibraryError):
        _lib.load(str(tmp_path / "nope.so"))


class TestHostConfig:
    def test_sensor_config_mirrors_reference_validation(self):
        with pytest.raises(InvalidArgumentError):
            SensorConfig(image_size=(0, 10))
        with pytest.raises(InvalidArgumentError):
            SensorConfig(image_size=(480, 640), sensing_area=(0.016, 0.013))
        assert SensorConfig().pixel_pitch == pytest.approx(2.5e-5)

    def test_marker_params_validation(self):
        with pytest.raises(InvalidArgumentError):
            MarkerParams(k_n=float("nan"))
        with pytest.raises(InvalidArgumentError):
            MarkerParams(lambda_s=0.0)

    def test_kernel_sizes(self):
        assert levels_from_kernel_sizes((1, 5)) == ((0.0, 0), (5 / 6.0, 2))
        for bad in ([4], [11, 5], []):
            with pytest.raises(InvalidArgumentError):
                levels_from_kernel_sizes(bad)

    def test_sigma_levels(self):
        assert levels_from_sigmas((1, 2, 4, 8)) == ((1.0, 3), (2.0, 6), (4.0, 12), (8.0, 24))
        with pytest.raises(InvalidArgumentError):
            levels_from_sigmas((-1.0,))

    def test_pipeline_config_shapes(self):
        s = SensorConfig.from_pitch(8, 10, 1e-4)
        with pytest.raises(InvalidArgumentError):
            PipelineConfig(s, ((1.0, 3),), np.zeros((2, 2, 3, 5)), np.zeros((8, 10, 3)))
        with pytest.raises(InvalidArgumentError):
            PipelineConfig(s, ((1.0, 3),), np.zeros((2, 2, 3, 6)), np.zeros((8, 9, 3)))
        cfg = PipelineConfig(s, ((1.0, 3),), np.zeros((2, 2, 3, 6)), np.zeros((8, 10, 3)))
        assert cfg.rest_grid.shape == (10, 10, 2)


# --------------------------------------------------------------------------- C layout
_FIELDS = {
    "tac_config": [f for f, _ in _lib.TacConfig._fields_],
    "tac_pipeline_args": [("in" if f == "in_" else f) for f, _ in _lib.TacPipelineArgs._fields_],
}


def _probe_source():
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "tac_b200.h"', "int main(void) {"]
    for st, fields in _FIELDS.items():
        lines.append(f'  printf("{st} size %zu\\n", sizeof({st}));')
        for f in fields:
            lines.append(f'  printf("{st} {f} %zu\\n", offsetof({st}, {f}));')
    lines += ["  return 0;", "}"]
    return "\n".join(lines) + "\n"


@pytest.fixture(scope="module")
def c_layout(tmp_path_factory):
    """Compile the header as strict C11 (-Werror) and read sizeof/offsetof."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc unavailable")
    d = tmp_path_factory.mktemp("clayout")
    (d / "probe.c").write_text(_probe_source())
    exe = d / "probe"
    cmd = ["gcc", "-std=c11", "-Wall", "-Wextra", "-Wpedantic", "-Werror", "-I", os.path.join(ROOT, "include"),
           str(d / "probe.c"), "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    layout = {}
    for line in out.splitlines():
        st, f, v = line.split()
        layout[(st, f)] = int(v)
    return layout


def _integration_binding():
    """Exec the reference-side ctypes snippet of INTEGRATION.md §2 (its CDLL
    pointed at the in-tree library)."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"```python\n(# tacsim/_b200\.py.*?)```", text, flags=re.S)
    assert m, "INTEGRATION.md lost its ctypes binding"
    code = m.group(1).replace('ctypes.CDLL("libtac_b200.so")', f"ctypes.CDLL({_lib.LIB_PATH!r})")
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


class TestCLayout:
    def test_header_is_valid_c11_and_cxx(self, tmp_path):
        import shutil
        import subprocess

        if shutil.which("g++") is None:
            pytest.skip("g++ unavailable")
        (tmp_path / "x.cc").write_text('#include "tac_b200.h"\nint main() { return sizeof(tac_config) > 0 ? 0 : 1; }\n')
        r = subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                            str(tmp_path / "x.cc"), "-o", str(tmp_path / "x")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr

    @pytest.mark.parametrize("name,cls", [("tac_config", _lib.TacConfig), ("tac_pipeline_args", _lib.TacPipelineArgs)])
    def test_package_binding_matches_compiled_layout(self, c_layout, name, cls):
        assert ctypes.sizeof(cls) == c_layout[(name, "size")]
        for (f, _), cf in zip(cls._fields_, _FIELDS[name]):
            assert getattr(cls, f).offset == c_layout[(name, cf)], f

    def test_integration_snippet_matches_compiled_layout(self, c_layout):
        ns = _integration_binding()
        for name, cls in (("tac_config", ns["TacConfig"]), ("tac_pipeline_args", ns["TacPipelineArgs"])):
            assert [f for f, _ in cls._fields_] == [f for f, _ in
                                                    (_lib.TacConfig if name == "tac_config" else _lib.TacPipelineArgs)._fields_]
            assert ctypes.sizeof(cls) == c_layout[(name, "size")]
            for (f, _), cf in zip(cls._fields_, _FIELDS[name]):
                assert getattr(cls, f).offset == c_layout[(name, cf)], (name, f)
        assert ns["TacConfig"]().struct_size == c_layout[("tac_config", "size")]

    def test_struct_size_mismatch_is_rejected(self):
        lib = _lib.load()
        c, keep = _cfg()
        c.struct_size = ctypes.sizeof(_lib.TacConfig) - 8  # a caller built against an older header
        h = ctypes.c_void_p()
        assert lib.tac_ctx_create(ctypes.byref(c), ctypes.byref(h)) == _lib.TAC_ERR_INVALID
        assert b"struct_size" in lib.tac_last_error()
        a = _lib.TacPipelineArgs()
        a.struct_size = 0
        assert lib.tac_pipeline(ctypes.c_void_p(1), ctypes.byref(a), None) == _lib.TAC_ERR_INVALID
        assert b"struct_size" in lib.tac_last_error()

    def test_execution_knobs_validated(self):
        lib = _lib.load()
        for field, val in (("lut_dtype", 7), ("kernel_path", 9), ("chunk_envs", -1)):
            c, keep = _cfg(**{field: val})
            h = ctypes.c_void_p()
            assert lib.tac_ctx_create(ctypes.byref(c), ctypes.byref(h)) == _lib.TAC_ERR_INVALID, field

    def test_library_reads_no_environment_knobs(self):
        """A/B switches live in tac_config, not in getenv."""
        data = open(_lib.LIB_PATH, "rb").read()
        for knob in (b"TAC_NO_TMA", b"TAC_LUT_ORDER", b"TAC_MAX_STRIP", b"TAC_FRAME", b"TAC_CHUNK"):
            assert knob + b"\0" not in data, knob
        src = "".join(open(os.path.join(ROOT, "paper_2411_04776_b200", "csrc", f)).read()
                      for f in os.listdir(os.path.join(ROOT, "paper_2411_04776_b200", "csrc"))
                      if f.endswith((".cu", ".cuh")))
        assert "getenv" not in src
