"""CPU-side checks of the C ABI (no GPU needed): the library loads, exports every symbol that
include/sasbp.h declares, and validates arguments before touching CUDA."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, cuda_available
import paper_2101_05888_b200 as pkg
from paper_2101_05888_b200 import sasbp


def _header_symbols():
    with open(os.path.join(ROOT, "include", "sasbp.h")) as f:
        txt = f.read()
    return set(re.findall(r"SASBP_API\s+[\w\s\*]+?\b(sas_\w+)\s*\(", txt))


@pytest.fixture(scope="module")
def lib():
    from paper_2101_05888_b200 import _build
    _build.build()
    return pkg.load_library()


def test_exports_match_header(lib):
    decl = _header_symbols()
    assert decl == set(sasbp.EXPORTS), decl ^ set(sasbp.EXPORTS)
    for name in decl:
        assert hasattr(lib, name), name


def test_version(lib):
    v = pkg.version()
    assert v.startswith("sasbp ") and "sm_100a" in v


def _grid(**kw):
    g = dict(origin=[0, 20, 0], step_x=[0.01, 0, 0], step_y=[0, 0.01, 0], step_z=[0, 0, 1.0], nx=64, ny=64, nz=1)
    g.update(kw)
    return sasbp.make_grid(g)


@pytest.mark.parametrize("args,grid_kw", [
    ((0.0, 30e3, 120e3, 1500.0), {}),                   # fc <= 0
    ((float("nan"), 30e3, 120e3, 1500.0), {}),          # non-finite fc
    ((120e3, 0.0, 120e3, 1500.0), {}),                  # bandwidth <= 0
    ((120e3, 200e3, 120e3, 1500.0), {}),                # bandwidth > fs
    ((120e3, 30e3, -1.0, 1500.0), {}),                  # fs <= 0
    ((120e3, 30e3, 120e3, 0.0), {}),                    # c <= 0
    ((120e3, 30e3, 120e3, 1500.0), {"nx": 0}),          # empty grid
    ((120e3, 30e3, 120e3, 1500.0), {"step_x": [0, 0, 0]}),                 # zero step
    ((120e3, 30e3, 120e3, 1500.0), {"step_y": [0.02, 0, 0]}),              # dependent steps
    ((120e3, 30e3, 120e3, 1500.0), {"origin": [float("inf"), 0, 0]}),      # non-finite origin
    ((120e3, 30e3, 120e3, 1500.0), {"nx": 65536, "ny": 65536}),            # > 2^31 pixels
])
def test_create_rejects_invalid(lib, args, grid_kw):
    g = _grid(**grid_kw)
    h = ctypes.c_void_p(123)
    st = lib.sas_bp_create(*args, ctypes.byref(g), ctypes.byref(h))
    assert st == sasbp.SAS_E_INVALID
    assert h.value is None
    assert lib.sas_last_error().decode() != ""


def test_create_null_pointers(lib):
    h = ctypes.c_void_p()
    assert lib.sas_bp_create(120e3, 30e3, 120e3, 1500.0, None, ctypes.byref(h)) == sasbp.SAS_E_INVALID
    g = _grid()
    assert lib.sas_bp_create(120e3, 30e3, 120e3, 1500.0, ctypes.byref(g), None) == sasbp.SAS_E_INVALID


@pytest.mark.skipif(cuda_available(), reason="checks the no-device path")
def test_create_without_device_is_unsupported(lib):
    g = _grid()
    h = ctypes.c_void_p()
    st = lib.sas_bp_create(120e3, 30e3, 120e3, 1500.0, ctypes.byref(g), ctypes.byref(h))
    assert st == sasbp.SAS_E_UNSUPPORTED
    with pytest.raises(sasbp.SasError):
        pkg.Backprojector(120e3, 30e3, 120e3, 1500.0, dict(origin=[0, 0, 0], step_x=[1, 0, 0], step_y=[0, 1, 0],
                                                          step_z=[0, 0, 1], nx=4, ny=4, nz=1))


def test_null_handle_calls(lib):
    lib.sas_bp_destroy(None)  # NULL-safe
    e = np.zeros(8, dtype=np.float32)
    d = np.zeros(3, dtype=np.float64)
    f32 = e.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    f64 = d.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    assert lib.sas_bp_set_pings(None, f32, 1, 1, 4, f64, f64, None) == sasbp.SAS_E_INVALID
    assert lib.sas_bp_form(None, f32) == sasbp.SAS_E_INVALID
    assert lib.sas_bp_form_device(None, None, None, 0) == sasbp.SAS_E_INVALID
    assert lib.sas_bp_count_terms(None, None, None) == sasbp.SAS_E_INVALID
    assert lib.sas_bp_form_streamed(None, f32, 1, 1, 4, f64, f64, None, f32, 0) == sasbp.SAS_E_INVALID
    assert lib.sas_bp_get_plan(None, None) == sasbp.SAS_E_INVALID
    assert lib.sas_bp_set_beam(None, None, None, 0) == sasbp.SAS_E_INVALID
    assert lib.sas_bp_set_motion(None, None, 0) == sasbp.SAS_E_INVALID
    assert lib.sas_bp_set_medium(None, 0.0, 1700.0) == sasbp.SAS_E_INVALID
    assert lib.sas_bp_workspace_bytes(None) == 0


def test_rangecompress_rejects_invalid(lib):
    x = np.zeros(16, dtype=np.float32)
    p = x.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    assert lib.sas_rangecompress(p, 1, 1, 0, p, 2, p) == sasbp.SAS_E_INVALID
    assert lib.sas_rangecompress(p, 1, 1, 4, p, 0, p) == sasbp.SAS_E_INVALID
    assert lib.sas_rangecompress(None, 1, 1, 4, p, 2, p) == sasbp.SAS_E_INVALID
    assert lib.sas_rangecompress_device(None, 1, 1, 4, None, 2, None, None) == sasbp.SAS_E_INVALID


def test_product_has_no_oracle_dependency():
    """The product package never imports the oracle."""
    pkg_dir = os.path.dirname(pkg.__file__)
    for dirpath, _, files in os.walk(pkg_dir):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                with open(os.path.join(dirpath, fn)) as f:
                    txt = f.read()
                assert "import oracle" not in txt and "oracle/" not in txt and "liboracle" not in txt, fn


def test_c_example_compiles_and_links_against_the_header():
    """include/sasbp.h is plain C11 and libsasbp.so resolves every symbol a C program uses
    (examples/c_smoke.c; it is run on the GPU by tests/test_c_example.py)."""
    import subprocess
    import tempfile
    out = os.path.join(tempfile.mkdtemp(), "c_smoke")
    r = subprocess.run(["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "c_smoke.c"), "-L", os.path.join(ROOT, "paper_2101_05888_b200"),
                        "-lsasbp", "-lm", "-Wl,-rpath," + os.path.join(ROOT, "paper_2101_05888_b200"), "-o", out],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
