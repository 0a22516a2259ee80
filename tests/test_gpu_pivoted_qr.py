"""GPU tests of qb_pivoted_qr (NEXT-4: QB -> partial pivoted QR): B P = Q~ R by
Householder QR with column pivoting on the GPU, Q^ = Q Q~.

Against the oracle's pivoted QR (oracle.qb.pivoted_qr: LAPACK dlaqp2's order written out, pinned
by hand-worked cases and against dgeqp3 in tests/test_oracle_qb.py) on the same B: the same
permutation (the first column of largest partial norm), R equal (same sign convention: beta =
-sign(alpha) ||x||), and the identities A P ~ Q^ R, Q^ orthonormal, |R(i,i)| non-increasing."""
import numpy as np
import pytest
import synth
from oracle import qb as oqb

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def qbmod():
    import paper_1503_07157_b200 as qbp
    from paper_1503_07157_b200 import build
    build.build()
    return qbp


def to_dev(A, dtype=np.float64):
    return torch.from_numpy(np.asfortranarray(A.astype(dtype))).cuda()


@pytest.mark.parametrize("m,n,kind,eps,b", [(600, 400, "exp10_20", 1e-6, 16), (1500, 900, "poly2", 1e-4, 64),
                                            (800, 2000, "exp_100", 1e-3, 100)])
def test_pivoted_qr_matches_oracle(qbmod, m, n, kind, eps, b):
    A = synth.make_matrix_np(m, n, synth.sigma(kind, min(m, n)), 91 + n)
    c = qbmod.QB(0)
    g = c.factor(to_dev(A), eps, b, 0, seed=2)
    k = g["k"]
    Q, B = g["Q"].cpu().numpy(), g["B"].cpu().numpy()
    r = c.pivoted_qr()
    c.close()
    perm, Qh, R = r["perm"], r["Qh"].cpu().numpy(), r["R"].cpu().numpy()
    Po, Qo, Ro = oqb.pivoted_qr(B)
    assert np.array_equal(perm, Po)
    assert np.allclose(np.tril(R, -1), 0.0)
    nB = np.linalg.norm(B)
    assert np.abs(R - Ro).max() <= 1e-12 * nB
    assert np.linalg.norm(Qh - Q @ Qo) <= 1e-11 * np.sqrt(k)
    assert np.all(np.diff(np.abs(np.diag(R))) <= 1e-12 * nB)
    assert np.abs(Qh.T @ Qh - np.eye(k)).max() <= 1e-12
    assert np.linalg.norm(Qh @ R - Q @ B[:, perm]) <= 1e-12 * nB
    assert np.linalg.norm(A[:, perm] - Qh @ R) <= eps * (1 + 1e-8)


def test_pivoted_qr_fp32_and_fixed_rank(qbmod):
    A = synth.make_matrix_np(3000, 400, synth.sigma("exp_100", 400), 5).astype(np.float32)
    c = qbmod.QB(0, dtype=qbmod.QB_F32)
    g = c.fixed_rank(to_dev(A, np.float32), 60, 1, seed=3)
    r = c.pivoted_qr()
    c.close()
    Q, B = g["Q"].double().cpu().numpy(), g["B"].double().cpu().numpy()
    Qh, R = r["Qh"].double().cpu().numpy(), r["R"].double().cpu().numpy()
    assert r["Qh"].dtype == torch.float32
    assert sorted(r["perm"].tolist()) == list(range(400))
    assert np.abs(Qh.T @ Qh - np.eye(60)).max() <= 1e-5
    assert np.linalg.norm(Qh @ R - Q @ B[:, r["perm"]]) <= 1e-5 * np.linalg.norm(B)


def test_pivoted_qr_without_factorization(qbmod):
    c = qbmod.QB(0)
    with pytest.raises(qbmod.QBError):
        c.pivoted_qr()
    c.close()


@pytest.mark.parametrize("env", ["QB_QRCP_NO_PERSIST", "QB_QRCP_LOOKAHEAD", "QB_QRCP_UNFUSED", "QB_QRCP_Q_UNBLOCKED"])
def test_pivoted_qr_other_schedules(qbmod, env):
    """The schedules the default one falls back to (multi-kernel blocked: too many columns per SM
    or too little shared memory) and the reference ones, each against the oracle in a fresh process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""), **{env: "1"})
    for case in (["1500", "900", "poly2", "1e-4", "64"], ["800", "2000", "exp_100", "1e-3", "100"]):
        p = subprocess.run([sys.executable, os.path.join(root, "tests", "qrcp_variant_check.py"), *case], env=e,
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stdout + p.stderr
