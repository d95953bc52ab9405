"""The C ABI from plain C on the GPU (-m gpu): examples/c_smoke.c images a point target through
libsasbp.so without Python and checks the peak lands on the target pixel."""
import os
import subprocess
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_example_focuses(require_gpu):
    from paper_2101_05888_b200 import _build
    _build.build()
    exe = os.path.join(tempfile.mkdtemp(), "c_smoke")
    lib = os.path.join(ROOT, "paper_2101_05888_b200")
    subprocess.run(["gcc", "-std=c11", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_smoke.c"), "-L", lib, "-lsasbp", "-lm", "-Wl,-rpath," + lib,
                    "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "peak" in r.stdout
