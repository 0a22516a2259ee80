"""GPU tests of rqb_svd (NEXT-1: QB -> partial SVD) through the C ABI.

  * the SPEC worked example (tests/golden: diag(3,2,1) embedded in 10x10 -> sigma = (3,2,1));
  * parity with the oracle's qb_to_svd on the oracle's own factorization of the same input:
    singular values within the QB-parity tolerance, U diag(S) V^T = Q B (the definition),
    U, V orthonormal, S descending; singular vectors compared up to sign where the gaps allow;
  * the tail rule (kkeep), k = 0, no-factorization error, FP32 context."""
import json
import os

import numpy as np
import pytest

import synth
from oracle import qb as oqb

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


@pytest.fixture(scope="module")
def qbmod():
    import paper_1503_07157_b200 as qbp
    from paper_1503_07157_b200 import build
    build.build()
    return qbp


def to_dev(A, dtype=np.float64):
    return torch.from_numpy(np.asfortranarray(A.astype(dtype))).cuda()


def test_svd_worked_example(qbmod):
    g = GOLD["qb_to_svd_diag321"]
    A = np.zeros((g["n"], g["n"]))
    A[0, 0], A[1, 1], A[2, 2] = g["d"]
    c = qbmod.QB(0)
    f = c.factor(to_dev(A), 0.0, g["ell"], 0, seed=2, kmax=g["ell"])
    s = c.svd()
    c.close()
    assert f["k"] == g["ell"]
    np.testing.assert_allclose(s["S"].cpu().numpy(), g["sigma"], atol=g["tol"])
    U, S, V = s["U"].cpu().numpy(), s["S"].cpu().numpy(), s["V"].cpu().numpy()
    assert np.linalg.norm(A - (U * S) @ V.T) < 1e-12


@pytest.mark.parametrize("m,n,kind,eps,b,q", [(400, 300, "exp10_20", 1e-6, 10, 0), (3000, 700, "exp_100", 1e-8, 64, 1),
                                              (1200, 2000, "poly2", 1e-4, 256, 0)])
def test_svd_parity_with_oracle(qbmod, m, n, kind, eps, b, q):
    A = synth.make_matrix_np(m, n, synth.sigma(kind, min(m, n)), 77 + m)
    nA = np.linalg.norm(A)
    o = oqb.randqb_pb(A, eps, b, q, seed=3)
    Uo, So, Vo = oqb.qb_to_svd(o.Q, o.B)
    c = qbmod.QB(0)
    f = c.factor(to_dev(A), eps, b, q, seed=3)
    s = c.svd()
    c.close()
    k = f["k"]
    assert k == o.k and k > 256 or k == o.k
    Q, B = f["Q"].cpu().numpy(), f["B"].cpu().numpy()
    U, S, V = s["U"].cpu().numpy(), s["S"].cpu().numpy(), s["V"].cpu().numpy()
    assert U.shape == (m, k) and S.shape == (k,) and V.shape == (n, k)
    assert (np.diff(S) <= 0).all() and (S >= 0).all()
    assert np.abs(U.T @ U - np.eye(k)).max() <= 1e-12
    assert np.abs(V.T @ V - np.eye(k)).max() <= 1e-12
    # the definition: U diag(S) V^T = Q B
    assert np.linalg.norm((U * S) @ V.T - Q @ B) <= 1e-13 * nA
    # parity with the oracle's SVD of its own factors (QB parity tolerance of the north_star)
    assert np.abs(S - So).max() <= 1e-10 * nA
    # leading singular vectors (well separated: relative gap > 1e-3) agree up to sign
    gaps = np.minimum(np.abs(np.diff(So, prepend=np.inf)), np.abs(np.diff(So, append=-np.inf)))
    for j in range(min(k, 20)):
        if gaps[j] > 1e-3 * So[0]:
            sgn = np.sign(U[:, j] @ Uo[:, j])
            assert np.abs(sgn * U[:, j] - Uo[:, j]).max() <= 1e-8
            assert np.abs(sgn * V[:, j] - Vo[:, j]).max() <= 1e-8


def test_svd_tail_rule_and_edges(qbmod):
    A = synth.make_matrix_np(500, 400, synth.sigma("exp10_20", 400), 5)
    c = qbmod.QB(0)
    with pytest.raises(qbmod.QBError):
        c.svd()                                   # no factorization yet
    f = c.factor(to_dev(A), 1e-6, 32, 0, seed=1)
    full = c.svd()
    part = c.svd(kkeep=20)
    assert part["U"].shape == (500, 20) and part["S"].shape == (20,) and part["V"].shape == (400, 20)
    assert torch.allclose(part["S"], full["S"][:20], rtol=0, atol=1e-14)
    assert torch.allclose(part["U"], full["U"][:, :20], rtol=0, atol=1e-12)
    assert torch.allclose(part["V"], full["V"][:, :20], rtol=0, atol=1e-12)
    # the tail rule's error: ||A - U_k' S_k' V_k'^T||_F^2 = ||A - QB||_F^2 + sum_{j > k'} S_j^2
    U, S, V = (part[x].cpu().numpy() for x in ("U", "S", "V"))
    lhs = np.linalg.norm(A - (U * S) @ V.T) ** 2
    rhs = f["resid"] ** 2 + float(np.sum(full["S"].cpu().numpy()[20:] ** 2))
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(A) ** 2
    # k = 0: empty triplets
    f0 = c.factor(to_dev(A), 1e6, 32, 0, seed=1)
    assert f0["k"] == 0
    e = c.svd()
    assert e["U"].shape == (500, 0) and e["S"].shape == (0,)
    c.close()


def test_svd_fp32_context(qbmod):
    A64 = synth.make_matrix_np(3000, 500, synth.sigma("exp_100", 500), 12)
    A32 = A64.astype(np.float32)
    c = qbmod.QB(0, dtype=qbmod.QB_F32)
    f = c.factor(to_dev(A32, np.float32), 1e-3, 64, 0, seed=2)
    s = c.svd()
    c.close()
    k = f["k"]
    U, S, V = (s[x].double().cpu().numpy() for x in ("U", "S", "V"))
    Q, B = f["Q"].double().cpu().numpy(), f["B"].double().cpu().numpy()
    assert s["U"].dtype == torch.float32
    assert np.abs(U.T @ U - np.eye(k)).max() <= 1e-5
    assert np.abs(V.T @ V - np.eye(k)).max() <= 1e-5
    assert np.linalg.norm((U * S) @ V.T - Q @ B) <= 1e-5 * np.linalg.norm(A64)
    np.testing.assert_allclose(S[:50], np.linalg.svd(Q @ B, compute_uv=False)[:50], rtol=1e-5)


@pytest.mark.parametrize("m,n,kind,eps,b", [(2500, 2200, "exp_150", 1e-4, 128), (1500, 1200, "poly2", 1e-5, 64)])
def test_svd_large_k_parity(qbmod, m, n, kind, eps, b):
    """k > 1024: many 32-column blocks in the Jacobi tournament, graded singular values spanning
    several decades (the tail of a QB factorization); parity with the oracle's LAPACK SVD of its
    own factors, orthonormal U and V, the definition U D V^T = QB."""
    A = synth.make_matrix_np(m, n, synth.sigma(kind, min(m, n)), 90 + m)
    nA = np.linalg.norm(A)
    o = oqb.randqb_pb(A, eps, b, 0, seed=4)
    Uo, So, Vo = oqb.qb_to_svd(o.Q, o.B)
    c = qbmod.QB(0)
    f = c.factor(to_dev(A), eps, b, 0, seed=4)
    s = c.svd()
    sweeps = qbmod.qb_svd_sweeps(c.ctx)
    c.close()
    k = f["k"]
    assert k == o.k and k >= 640
    Q, B = f["Q"].cpu().numpy(), f["B"].cpu().numpy()
    U, S, V = s["U"].cpu().numpy(), s["S"].cpu().numpy(), s["V"].cpu().numpy()
    assert (np.diff(S) <= 0).all() and S[-1] > 0
    assert np.abs(U.T @ U - np.eye(k)).max() <= 1e-12
    assert np.abs(V.T @ V - np.eye(k)).max() <= 1e-12
    assert np.linalg.norm((U * S) @ V.T - Q @ B) <= 1e-13 * nA
    assert np.abs(S - So).max() <= 1e-10 * nA
    assert 1 <= sweeps <= 20


def test_svd_eps_tail_rule(qbmod):
    """rqb_svd(eps): the rank kept is the tail rule's (oracle.tail_rank on the oracle's own
    factorization: ||A - U_k' D_k' V_k'^T||^2 = ||A - QB||^2 + sum_{j > k'} D_j^2 <= eps^2,
    PAPER.md:398-406), and the truncated triplets meet eps against the pristine A."""
    A = synth.make_matrix_np(900, 700, synth.sigma("exp10_20", 700), 8)
    o = oqb.randqb_pb(A, 1e-6, 32, 0, seed=1)
    _, So, _ = oqb.qb_to_svd(o.Q, o.B)
    c = qbmod.QB(0)
    f = c.factor(to_dev(A), 1e-6, 32, 0, seed=1)
    assert f["k"] == o.k
    for eps in (1e-6, 1e-4, 1e-2, 10.0):
        kk_o = oqb.tail_rank(So, o.hist[-1][2], eps)
        s = c.svd(eps=eps)
        assert s["kk"] == kk_o, (eps, s["kk"], kk_o)
        if kk_o > 0:
            U, S, V = s["U"].cpu().numpy(), s["S"].cpu().numpy(), s["V"].cpu().numpy()
            assert np.linalg.norm(A - (U * S) @ V.T) <= eps * (1 + 1e-8)
    s = c.svd(eps=1e-4, kkeep=5)       # both: the smaller rank
    assert s["kk"] == 5
    with pytest.raises(qbmod.QBError):
        c.svd(eps=-1.0)
    c.close()


def test_svd_preconditioned_and_plain_in_fresh_processes():
    """rqb_svd with and without the QR preconditioning step (QB_SVD_PRECOND=1 / 0; the default depends
    on k), each against the oracle's SVD of the same QB in a fresh process (the variable is read once
    per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import numpy as np, torch, synth
from oracle import qb as oqb
import paper_1503_07157_b200 as qbp
A = synth.make_matrix_np(1500, 1200, synth.sigma("exp_150", 1200), 77)
c = qbp.QB(0)
g = c.factor(torch.from_numpy(np.asfortranarray(A)).cuda(), 1e-6, 128, 0, seed=5)
Q, B = g["Q"].cpu().numpy(), g["B"].cpu().numpy()
s = c.svd()
U, S, V = s["U"].cpu().numpy(), s["S"].cpu().numpy(), s["V"].cpu().numpy()
So = np.linalg.svd(B, compute_uv=False)
nA = np.linalg.norm(A)
assert np.abs(S - So[:len(S)]).max() <= 1e-10 * nA
assert np.linalg.norm(U * S @ V.T - Q @ B) <= 1e-13 * nA
assert np.abs(U.T @ U - np.eye(len(S))).max() <= 1e-12 and np.abs(V.T @ V - np.eye(len(S))).max() <= 1e-12
print("ok", g["k"], len(S))
'''
    for v in ("0", "1"):
        e = dict(os.environ, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""), QB_SVD_PRECOND=v)
        p = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=300, cwd=root)
        assert p.returncode == 0, p.stdout + p.stderr
