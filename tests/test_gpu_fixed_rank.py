"""GPU parity of the fixed-rank schemes (NEXT-4): randQB (Fig. 1) and randQB_p
(Fig. 3), unblocked, through qb_fixed_rank, against the oracle's randqb /
randqb_p on the same seeded inputs (Ω columns 0..l-1 of the same generator).

Tolerances as for qb_factor (north_star FP64): ||Q^T Q - I||_max <= 1e-12, ||Q_g B_g - Q_o B_o||_F
<= 1e-10 ||A||_F, the reported residual = the true one.  Widths above 256 exercise the blocked orth
(block Gram-Schmidt + CholeskyQR2 per 256 columns)."""
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


@pytest.fixture(scope="module")
def ctx(qbmod):
    c = qbmod.QB(0)
    yield c
    c.close()


def to_dev(A, dtype=np.float64):
    return torch.from_numpy(np.asfortranarray(A.astype(dtype))).cuda()


def check(A, g, Qo, Bo, tol_orth=1e-12, tol_qb=1e-10):
    nA = np.linalg.norm(A)
    Q, B = g["Q"].double().cpu().numpy(), g["B"].double().cpu().numpy()
    l = Q.shape[1]
    assert np.abs(Q.T @ Q - np.eye(l)).max() <= tol_orth
    diff = np.hstack([Q, Qo]) @ np.vstack([B, -Bo])
    assert np.linalg.norm(diff) <= tol_qb * nA, np.linalg.norm(diff) / nA
    true = np.linalg.norm(A - Q @ B)
    if g["resid"] is not None:
        assert abs(g["resid"] - true) <= 1e-12 * nA + 1e-8 * true
    return true


@pytest.mark.parametrize("m,n,l,kind", [(600, 400, 60, "exp_100"), (1000, 800, 300, "poly2"),
                                        (300, 1200, 100, "exp_100"), (2000, 600, 520, "exp_150")])
@pytest.mark.parametrize("P", [0, 1, 2])
def test_fixed_rank_parity(qbmod, ctx, m, n, l, kind, P):
    A = synth.make_matrix_np(m, n, synth.sigma(kind, min(m, n)), 40 + m + l)
    Qo, Bo = oqb.randqb_p(A, l, P, seed=5) if P > 0 else oqb.randqb(A, l, seed=5)
    g = ctx.fixed_rank(to_dev(A), l, P, seed=5)
    check(A, g, Qo, Bo)


def test_blocked_equals_unblocked(qbmod, ctx):
    """Fig. 2 with b < l and eps = 0, kmax = l spans the same space as Fig. 1 with the same Ω
    (the Ω_i are slices of Ω, eq. (OmegaBlock) :479-484)."""
    A = synth.make_matrix_np(800, 500, synth.sigma("exp_100", 500), 3)
    l = 96
    f = ctx.fixed_rank(to_dev(A), l, 0, seed=9)
    b = ctx.factor(to_dev(A), 0.0, 32, 0, seed=9, kmax=l)
    assert b["k"] == l
    Qf, Bf = f["Q"].cpu().numpy(), f["B"].cpu().numpy()
    Qb, Bb = b["Q"].cpu().numpy(), b["B"].cpu().numpy()
    assert np.linalg.norm(Qf @ Bf - Qb @ Bb) <= 1e-10 * np.linalg.norm(A)


def test_skip_power_orth_variant(qbmod, ctx):
    """PAPER.md:919-927 unblocked: Y = A (A^* A)^P Ω, orth once — against the oracle's variant."""
    A = synth.make_matrix_np(700, 500, synth.sigma("exp_100", 500), 11)
    l = 40
    Qo, Bo = oqb.randqb_p(A, l, 1, seed=2, skip_power_orth=True)
    g = ctx.fixed_rank(to_dev(A), l, 1, seed=2, flags=qbmod.QB_SKIP_POWER_ORTH)
    check(A, g, Qo, Bo, tol_qb=1e-9)


def test_fixed_rank_then_svd_and_errors(qbmod, ctx):
    A = synth.make_matrix_np(500, 400, synth.sigma("poly2", 400), 21)
    g = ctx.fixed_rank(to_dev(A), 50, 1, seed=4)
    s = ctx.svd()
    Q, B = g["Q"].cpu().numpy(), g["B"].cpu().numpy()
    np.testing.assert_allclose(s["S"].cpu().numpy(), np.linalg.svd(Q @ B, compute_uv=False)[:50],
                               rtol=0, atol=1e-12 * np.linalg.norm(A))
    for bad in [dict(l=401), dict(l=0), dict(P=-1)]:
        kw = dict(l=10, P=0)
        kw.update(bad)
        with pytest.raises(qbmod.QBError):
            ctx.fixed_rank(to_dev(A), kw["l"], kw["P"])


def test_fixed_rank_overwrite_leaves_residual(qbmod, ctx):
    A = synth.make_matrix_np(400, 300, synth.sigma("exp_100", 300), 8)
    Ad = to_dev(A)
    g = ctx.fixed_rank(Ad, 64, 0, seed=1, overwrite=True)
    Q, B = g["Q"].cpu().numpy(), g["B"].cpu().numpy()
    assert np.abs(Ad.cpu().numpy() - (A - Q @ B)).max() <= 1e-13 * np.abs(A).max() * 64
    assert abs(g["resid"] - np.linalg.norm(A - Q @ B)) <= 1e-12 * np.linalg.norm(A)


@pytest.mark.parametrize("P", [0, 1])
def test_fixed_rank_fp32(qbmod, P):
    """FP32 context (3xTF32 tensor-core products, FP64 orth): FP32 tolerances of the north_star."""
    A64 = synth.make_matrix_np(3000, 500, synth.sigma("exp_100", 500), 17)
    A32 = A64.astype(np.float32)
    Aw = A32.astype(np.float64)
    if P > 0:
        Qo, Bo = oqb.randqb_p(Aw, 100, P, seed=6, omega_dtype=np.float32)
    else:
        Qo, Bo = oqb.randqb(Aw, 100, seed=6, omega_dtype=np.float32)
    c = qbmod.QB(0, dtype=qbmod.QB_F32)
    g = c.fixed_rank(to_dev(A32, np.float32), 100, P, seed=6)
    c.close()
    assert g["Q"].dtype == torch.float32
    check(Aw, g, Qo, Bo, tol_orth=1e-5, tol_qb=1e-4)
