"""Host-side checks of bench.py (the driver contract): --gpus N never silently runs one rank,
and the algorithmic work / byte counts follow SURVEY.md §8(d) (PAPER.md:902 cost model)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_gpus_n_without_enough_devices_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has >= 2 GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    assert "needs 2 visible GPUs" in r.stderr
    assert r.stdout.strip() == ""          # no JSON line claiming a result


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], capture_output=True,
                       text=True, env=env, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_falg_matches_the_cost_model():
    # T, q = 0, k = 2816 (11 blocks of 256): 3 GEMM passes of 2mnk + re-projection 2mk(k-b)
    # + Householder-equivalent orth 2 * 4 m b^2 per block (7.162 TFLOP)
    F = bench.falg(20000, 20000, 2816, 256, 0, 11)
    assert abs(F / 1e12 - 7.162) < 0.01
    # one block, no re-projection, q = 1: 5 passes + 3 orth calls of 4 m b^2 and one 4 n b^2
    m, n, b = 100, 80, 10
    assert bench.falg(m, n, b, b, 1, 1) == 5 * 2 * m * n * b + 3 * 4 * m * b * b + 4 * n * b * b


def test_bytes_alg():
    m, n, b, es = 1000, 500, 10, 8
    # two blocks, q = 0: 3 passes over A per block + 2 m ell_{i-1} es for the second block
    assert bench.bytes_alg(m, n, 20, b, 0, 2, es) == 2 * 3 * m * n * es + 2 * m * 10 * es
