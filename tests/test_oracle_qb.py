"""Pins for the oracle's QB loop (oracle/qb.py) against what the paper and the mathematics
fix — not against a retyped copy of the oracle.  Each test names the passage it checks
(PAPER.md line numbers; SPEC.md worked examples via tests/golden/)."""
import json
import os

import numpy as np
import pytest

import synth
from oracle import qb

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))
U64 = np.finfo(np.float64).eps / 2


def small_matrix(m=200, n=150, kind="inv", seed=0):
    r = min(m, n)
    if kind == "inv":
        sig = 1.0 / np.arange(1, r + 1)
    elif kind == "exp10_25":
        sig = 10.0 ** (-np.arange(1, r + 1) / 25.0)
    else:
        sig = synth.sigma(kind, r)
    return synth.make_matrix_np(m, n, sig, seed), sig


# ---------------------------------------------------------------- primitives
def test_frobenius_worked_example():
    g = GOLD["frobenius"]
    assert qb.frob2(np.array(g["X"])) == g["norm"] ** 2


def test_orth_worked_example():
    g = GOLD["orth_2x1"]
    Q = qb.orth(np.array(g["X"]))
    np.testing.assert_allclose(Q, np.array(g["Q"]), rtol=0, atol=1e-15)


def test_orth_closed_form_gram_schmidt():
    # columns x1 = (1,0,1), x2 = (1,1,0): q1 = x1/sqrt2, q2 = (1/2, 1, -1/2)/sqrt(3/2) by hand
    X = np.array([[1.0, 1.0], [0.0, 1.0], [1.0, 0.0]])
    Q = qb.orth(X)
    q1 = np.array([1.0, 0.0, 1.0]) / np.sqrt(2.0)
    q2 = np.array([0.5, 1.0, -0.5]) / np.sqrt(1.5)
    np.testing.assert_allclose(Q[:, 0], q1, atol=1e-15)
    np.testing.assert_allclose(Q[:, 1], q2, atol=1e-15)


def test_orth_is_orthonormal_basis_of_range():
    X = np.random.default_rng(1).standard_normal((300, 40))
    Q = qb.orth(X)
    assert np.abs(Q.T @ Q - np.eye(40)).max() < 1e-14
    # X = Q (Q^T X): ran(X) inside ran(Q)
    assert np.linalg.norm(X - Q @ (Q.T @ X)) < 1e-13 * np.linalg.norm(X)
    # diag(R) >= 0 convention (reading R7): Q^T X is upper triangular with positive diagonal
    R = Q.T @ X
    assert np.all(np.diag(R) > 0)
    assert np.abs(np.tril(R, -1)).max() < 1e-13


def test_optimal_error_worked_example():
    g = GOLD["optimal_errors"]
    for case in g["cases"]:
        assert abs(synth.optimal_error(np.array(g["d"]), case["k"]) - case["frobenius"]) < 1e-15


def test_qb_to_svd_worked_example():
    g = GOLD["qb_to_svd_diag321"]
    A = np.zeros((g["n"], g["n"]))
    A[0, 0], A[1, 1], A[2, 2] = g["d"]
    r = qb.randqb_pb(A, eps=0.0, b=g["ell"], q=0, seed=2, kmax=g["ell"])
    U, D, V = qb.qb_to_svd(r.Q, r.B)
    np.testing.assert_allclose(D, g["sigma"], atol=g["tol"])
    assert np.linalg.norm(A - (U * D) @ V.T) < 1e-12


# ---------------------------------------------------------------- the blocked loop
@pytest.mark.parametrize("q", [0, 1, 2])
def test_relations_and_proposition_1(q):
    """Prop. 1 and eq. (QB_alg_relations1) (:116-121):
    Q̄ orthonormal; A^(i) = (I - Q̄Q̄^*)A; B̄ = Q̄^*A — checked after every block by rerunning
    with kmax = ell_i (the loop is deterministic in (seed, b))."""
    A, _ = small_matrix()
    nA = np.linalg.norm(A)
    full = qb.randqb_pb(A, eps=1e-3, b=10, q=q, seed=4)
    for ell, w, r2, ei in full.hist:
        r = qb.randqb_pb(A, eps=0.0, b=10, q=q, seed=4, kmax=ell)
        assert r.k == ell
        assert np.abs(r.Q.T @ r.Q - np.eye(ell)).max() < 1e-13
        np.testing.assert_allclose(r.B, r.Q.T @ A, atol=1e-13 * nA)
        resid = A - r.Q @ r.B
        assert np.linalg.norm(resid - (A - r.Q @ (r.Q.T @ A))) < 1e-13 * nA
        # the recorded r2 is the directly computed ||A^(i)||_F^2
        assert abs(np.sqrt(r2) - np.linalg.norm(resid)) < 1e-13 * nA


def test_range_property_prop1c():
    """R(Q̄_i) = R(Ȳ_i), Ȳ_i = [AΩ_1 ... AΩ_i] with the ORIGINAL A, q = 0."""
    A, _ = small_matrix(kind="exp10_25")
    r = qb.randqb_pb(A, eps=0.0, b=8, q=0, seed=5, kmax=32)
    Ybar = A @ qb.omega(5, A.shape[1], 0, 32)
    Qy = qb.orth(Ybar)
    assert np.linalg.norm(Qy @ Qy.T - r.Q @ r.Q.T, 2) < 1e-8


@pytest.mark.parametrize("b", [5, 10, 20])
def test_blocked_equals_unblocked_projector(b):
    """for the same Ω the blocked projector equals the unblocked one,
    so A - QQ^*A agrees with randQB (Fig. 1).  SPEC.md:621 asks 1e-10 ||A||."""
    A, _ = small_matrix()
    ell = 60
    r = qb.randqb_pb(A, eps=0.0, b=b, q=0, seed=8, kmax=ell)
    Qt, Bt = qb.randqb(A, ell, seed=8)
    assert np.linalg.norm((A - r.Q @ r.B) - (A - Qt @ Bt)) < 1e-10 * np.linalg.norm(A)


def test_power_step_single_block():
    """Fig. 4 with one block equals Fig. 3 (randQB_p) with ℓ = b, and its
    range is that of (AA^*)^P AΩ when that matrix is well conditioned."""
    A, _ = small_matrix(kind="inv")
    for P in (1, 2):
        r = qb.randqb_pb(A, eps=0.0, b=12, q=P, seed=3, kmax=12)
        Qp, Bp = qb.randqb_p(A, 12, P, seed=3)
        assert np.linalg.norm(r.Q @ r.Q.T - Qp @ Qp.T, 2) < 1e-12
        Y = A @ qb.omega(3, A.shape[1], 0, 12)
        for _ in range(P):
            Y = A @ (A.T @ Y)
        Qy = qb.orth(Y)
        assert np.linalg.norm(r.Q @ r.Q.T - Qy @ Qy.T, 2) < 1e-6


def test_power_steps_sharpen_accuracy():
    """σ^(2P+1) decay: for a fixed rank, q = 1 is closer to optimal."""
    A, sig = small_matrix(kind="inv")
    r0 =qb.randqb_pb(A, 0.0, 10, 0, 1, kmax=40)
    r1 = qb.randqb_pb(A, 0.0, 10, 1, 1, kmax=40)
    opt = synth.optimal_error(sig, 40)
    e0 = np.linalg.norm(A - r0.Q @ r0.B)
    e1 = np.linalg.norm(A - r1.Q @ r1.B)
    assert opt <= e1 < e0
    assert e1 < 1.2 * opt


@pytest.mark.parametrize("cfg_q", [("C1", 0), ("C1", 1)])
def test_stop_rule_eckart_young_and_identity(cfg_q):
    """C1 (BASELINE configs[0]): stop rule (Fig. 2 line (6)), Eckart-Young floor
    (PAPER.md:229-239), k >= k_eps, and the Frobenius identity ||A-QB||^2 = ||A||^2 - ||B||^2
    within 6 u ||A||^2 (reading R1)."""
    name, q = cfg_q
    cfg = synth.CONFIGS[name]
    sig = synth.config_sigma(cfg)
    A = synth.make_matrix_np(cfg.m, cfg.n, sig, cfg.seed_matrix)
    r = qb.randqb_pb(A, cfg.eps, cfg.b, q, cfg.seed_omega)
    true = np.linalg.norm(A - r.Q @ r.B)
    assert r.status == qb.QB_OK
    assert true <= cfg.eps * (1 + 1e-8)
    assert r.k % cfg.b == 0
    # the block before did not meet the tolerance
    assert r.hist[-2][2] > cfg.eps ** 2
    # Eckart-Young: no rank-k factorisation beats the tail of the spectrum
    kq = synth.eps_rank(sig, cfg.eps)
    assert r.k >= kq
    assert true >= synth.optimal_error(sig, r.k) * (1 - 1e-8)
    if q >= 1:  # soft check of the north_star "k within b of the ε-rank" (reading R20)
        assert r.k <= -(-kq // cfg.b) * cfg.b + cfg.b
    nA2 = qb.frob2(A)
    for ell, w, r2, ei in r.hist:
        assert abs(ei - r2) <= 6 * U64 * nA2
    # monotone residual history
    r2s = [h[2] for h in r.hist]
    assert all(x >= y for x, y in zip(r2s, r2s[1:]))


def test_brute_force_svd_tiny():
    """On tiny inputs the true ε-rank from a full SVD (LAPACK) bounds k from below and the
    residual from below (Eckart-Young)."""
    rng = np.random.default_rng(12)
    for trial in range(5):
        A = rng.standard_normal((30, 20)) @ np.diag(0.5 ** np.arange(20)) @ rng.standard_normal((20, 20))
        s = np.linalg.svd(A, compute_uv=False)
        eps = 1e-3 * s[0]
        r = qb.randqb_pb(A, eps, b=3, q=1, seed=trial)
        kq = synth.eps_rank(s, eps)
        assert kq <= r.k <= 20
        assert np.linalg.norm(A - r.Q @ r.B) >= np.sqrt(np.sum(s[r.k:] ** 2)) * (1 - 1e-10)
        assert np.linalg.norm(A - r.Q @ r.B) <= eps * (1 + 1e-8)


def test_reprojection_keeps_orthogonality():
    """Line (3'): without it the blocks drift into the earlier span;
    with it ||Q^*Q - I|| stays at round-off."""
    A, _ = small_matrix(1000, 800, kind="exp10_25", seed=3)
    with_ = qb.randqb_pb(A, 1e-13, b=20, q=0, seed=1)
    without = qb.randqb_pb(A, 1e-13, b=20, q=0, seed=1, reproj=False)
    o_with = np.abs(with_.Q.T @ with_.Q - np.eye(with_.k)).max()
    o_without = np.abs(without.Q.T @ without.Q - np.eye(without.k)).max()
    assert o_with < 1e-13
    assert o_without > 1e3 * o_with


def test_degenerate_inputs():
    A = np.zeros((20, 10))
    r = qb.randqb_pb(A, 1e-8, 4)
    assert (r.status, r.k) == (qb.QB_OK, 0)
    A = np.random.default_rng(0).standard_normal((20, 10))
    r = qb.randqb_pb(A, 10 * np.linalg.norm(A), 4)   # reading R3: checked before block 1
    assert (r.status, r.k) == (qb.QB_OK, 0)
    r = qb.randqb_pb(A, 0.0, 4, kmax=6)              # reading R5: narrowed last block
    assert (r.status, r.k) == (qb.QB_NOT_CONVERGED, 6)
    assert [h[1] for h in r.hist] == [4, 2]
    r = qb.randqb_pb(A, 1e-10, 4)                    # full rank: exhausts at min(m, n)
    assert r.k == 10 and r.resid < 1e-10


def test_empty_inputs():
    """m = 0 or n = 0: ||A||_F = 0 <= eps for every eps >= 0, so k = 0 (reading R3)."""
    for shape in ((0, 7), (7, 0), (0, 0)):
        r = qb.randqb_pb(np.zeros(shape), 0.0, 4)
        assert (r.status, r.k) == (qb.QB_OK, 0)
        assert r.Q.shape == (shape[0], 0) and r.B.shape == (0, shape[1])


def test_rank_exhaustion_inside_a_block():
    """Exact rank 25 with b = 10: the third block's sketch has rank 5; orth (Householder)
    still returns an orthonormal block and the residual reaches round-off (reading R8)."""
    rng = np.random.default_rng(2)
    A = rng.standard_normal((120, 25)) @ rng.standard_normal((25, 90))
    r = qb.randqb_pb(A, 1e-9 * np.linalg.norm(A), 10, q=0, seed=3)
    assert r.k == 30
    assert np.abs(r.Q.T @ r.Q - np.eye(30)).max() < 1e-13
    assert np.linalg.norm(A - r.Q @ r.B) < 1e-12 * np.linalg.norm(A)


def test_matrix1_rank_about_75():
    """Matrix 1 (d_j = g_j^2 0.65^(j-1)) has rank about 75 to precision
    1e-15; the adaptive scheme with q = 1 stops within a block or two of that rank."""
    g = GOLD["matrix1_rank"]
    rng = np.random.default_rng(1049)
    r = min(g["m"], g["n"])
    d = rng.random(r) ** 2 * g["beta"] ** np.arange(r)
    lo, hi = g["rank_range"]
    assert lo <= int(np.sum(d > g["precision"])) <= hi
    A = synth.make_matrix_np(g["m"], g["n"], d, 7)
    res = qb.randqb_pb(A, 1e-14, 5, q=1, seed=1)
    kq = synth.eps_rank(d, 1e-14)
    assert kq <= res.k <= kq + 10
    assert lo <= res.k <= hi


@pytest.mark.parametrize("P,floor", [(1, 1e-5), (2, 1e-3)])
def test_skip_power_orth_floors(P, floor):
    """PAPER.md:1170-1182 (Fig. 'skipqr' caption and Remark): without re-orthonormalisation
    between applications of A and A^*, the unblocked scheme cannot resolve beyond
    sigma_1 eps_mach^(1/(2P+1)) (1e-5 for P = 1, 1e-3 for P = 2), while the blocked scheme
    "always reaches full precision"."""
    r = 400
    sig = 10.0 ** (-np.arange(1, r + 1) / 25.0)
    A = synth.make_matrix_np(600, 400, sig, 3)
    opt = synth.optimal_error(sig, 200)
    Qu, Bu = qb.randqb_p(A, 200, P, seed=1, skip_power_orth=True)
    eu = np.linalg.norm(A - Qu @ Bu)
    assert 0.1 * floor <= eu <= 10 * floor            # stuck at the predicted floor
    Qo, Bo = qb.randqb_p(A, 200, P, seed=1)
    assert np.linalg.norm(A - Qo @ Bo) <= 1.2 * opt   # with orth: near-optimal
    rb = qb.randqb_pb(A, 0.0, 20, P, seed=1, kmax=200, skip_power_orth=True)
    assert np.linalg.norm(A - rb.Q @ rb.B) <= 1.2 * opt  # blocked, no orth: full precision
    # q = 0: the variant is the plain scheme
    r0 = qb.randqb_pb(A, 0.0, 20, 0, seed=1, kmax=60, skip_power_orth=True)
    r1 = qb.randqb_pb(A, 0.0, 20, 0, seed=1, kmax=60)
    assert np.array_equal(r0.Q, r1.Q)


def test_tail_rank_worked_example():
    """diag(3, 2, 1) with an exact QB (resid 0): dropping sigma = 1 costs 1, dropping 2 as well 5
    (the SVD tail identity); eps = 1.5 keeps 2 triplets, eps^2 = 5 (<=, reading R4) keeps 1,
    kkeep caps, eps = 0 keeps all."""
    D = np.array([3.0, 2.0, 1.0])
    assert qb.tail_rank(D, 0.0, 1.5) == 2
    assert qb.tail_rank(D, 0.0, np.sqrt(5.0) * (1 + 1e-12)) == 1
    assert qb.tail_rank(D, 0.0, 0.999) == 3
    assert qb.tail_rank(D, 0.0, 100.0) == 0
    assert qb.tail_rank(D, 0.0, 1.5, kkeep=1) == 1
    assert qb.tail_rank(D, 0.0, 0.0) == 3
    assert qb.tail_rank(D, 1.25, 1.5) == 2       # resid^2 + 1 = 2.25 <= eps^2 = 2.25: drop sigma = 1
    assert qb.tail_rank(D, 1.2500001, 1.5) == 3  # 2.2500001 > 2.25: keep all


def test_truncated_svd_error_identity():
    """||A - U_k' D_k' V_k'^*||_F^2 = ||A - QB||_F^2 + sum_{j >= k'} D_j^2 for every k' (the
    factorization's Q is orthonormal and the SVD of B is exact up to rounding)."""
    A = synth.make_matrix_np(300, 240, synth.sigma("exp10_20", 240), 9)
    r = qb.randqb_pb(A, 1e-5, 16)
    U, D, V = qb.qb_to_svd(r.Q, r.B)
    resid2 = r.hist[-1][2]
    nA2 = qb.frob2(A)
    for kk in (0, 5, 37, len(D)):
        lhs = qb.frob2(A - (U[:, :kk] * D[:kk]) @ V[:, :kk].T)
        assert abs(lhs - (resid2 + float(np.sum(D[kk:] ** 2)))) <= 1e-13 * nA2
    eps = np.sqrt(resid2 + np.sum(D[60:] ** 2)) * (1 + 1e-9)
    Ut, Dt, Vt = qb.qb_to_svd_truncated(r.Q, r.B, resid2, eps)
    assert len(Dt) == 60 and Ut.shape == (300, 60) and Vt.shape == (240, 60)
    assert qb.frob2(A - (Ut * Dt) @ Vt.T) <= eps ** 2 * (1 + 1e-9)


def test_pivoted_qr_hand_examples():
    """Two cases worked by hand from LAPACK dlaqp2's definitions:
    B = [[3, 1], [4, 2]]: no pivoting, alpha = 3, ||x|| = 5, beta = -5, tau = 1.6, v = (1, 0.5),
    column 2 -> (1, 2) - 1.6 * 2 * (1, 0.5) = (-2.2, 0.4); the last reflector is trivial (tau = 0).
    B = [[1, 0, 2], [0, 3, 0]]: pivot column 1 (norm 3), alpha = 0 -> beta = -3, tau = 1, v = (1, 1);
    the trailing columns become (0, -1) and (0, -2), so step 2 pivots original column 2."""
    perm, Q, R = qb.pivoted_qr(np.array([[3.0, 1.0], [4.0, 2.0]]))
    assert list(perm) == [0, 1]
    np.testing.assert_allclose(R, [[-5.0, -2.2], [0.0, 0.4]], atol=1e-15)
    perm, Q, R = qb.pivoted_qr(np.array([[1.0, 0.0, 2.0], [0.0, 3.0, 0.0]]))
    assert list(perm) == [1, 2, 0]
    np.testing.assert_allclose(R, [[-3.0, 0.0, 0.0], [0.0, -2.0, -1.0]], atol=1e-15)
    np.testing.assert_allclose(Q, [[0.0, -1.0], [-1.0, 0.0]], atol=1e-15)


@pytest.mark.parametrize("shape", [(40, 70), (64, 64), (30, 200)])
def test_pivoted_qr_matches_lapack_and_invariants(shape):
    """An independent implementation (LAPACK dgeqp3 through scipy) picks the same permutation and
    the same R up to row signs; B P = Q~ R, Q~ orthogonal, |R_ii| non-increasing."""
    import scipy.linalg
    l, n = shape
    rng = np.random.default_rng(l + n)
    B = (rng.standard_normal((l, n)) * np.exp(-np.arange(n) / 30.0)[None, :])[:, rng.permutation(n)]
    perm, Q, R = qb.pivoted_qr(B)
    Ql, Rl, pl = scipy.linalg.qr(B, mode="economic", pivoting=True)
    assert list(perm[:min(l, n)]) == list(pl[:min(l, n)])
    s = np.sign(np.diag(R)) * np.sign(np.diag(Rl))
    np.testing.assert_allclose(s[:, None] * R[:min(l, n)], Rl, atol=1e-12 * np.linalg.norm(B))
    np.testing.assert_allclose(B[:, perm], Q @ R, atol=1e-12 * np.linalg.norm(B))
    np.testing.assert_allclose(Q.T @ Q, np.eye(l), atol=1e-13)
    d = np.abs(np.diag(R))
    assert (np.diff(d) <= 1e-12 * d[0]).all()
