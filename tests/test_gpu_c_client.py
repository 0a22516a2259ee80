"""The C ABI from plain C (no Python, no CUDA headers): examples/qb_example.c is compiled with gcc
against include/qb.h and libqb.so and run on the GPU (qb_factor_host, a host-side residual check,
rqb_svd)."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_client(tmp_path):
    from paper_1503_07157_b200 import build
    lib = build.build()
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = tmp_path / "qb_example"
    libdir = os.path.dirname(lib)
    subprocess.run(["gcc", "-O2", "-std=c99", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "qb_example.c"), "-L", libdir, "-l:libqb.so",
                    f"-Wl,-rpath,{libdir}", "-lm", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "k = " in r.stdout and "rqb_svd" in r.stdout
