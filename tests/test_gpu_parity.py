"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded inputs.

Tolerances are the north_star's (BASELINE.json), FP64: identical k outside the tie zone
(reading R19), ||Q^*Q - I||_max <= 1e-12, ||Q_g B_g - Q_o B_o||_F / ||A||_F <= 1e-10 (one
GEMM [Q_g Q_o][B_g; -B_o], reading in DESIGN.md §6), ||A - Q_g B_g||_F <= eps (1 + 1e-8).
Ω is compared bit for bit."""
import numpy as np
import pytest

import synth
from oracle import omega as oomega
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


def to_dev(A):
    return torch.from_numpy(np.asfortranarray(A)).cuda()  # Fortran order -> stride(0) == 1


def in_tie_zone(res_o, eps, rel=1e-8):
    return any(abs(np.sqrt(h[2]) - eps) <= rel * eps for h in res_o.hist)


def check_parity(A, g, o, eps, tol_orth=1e-12, tol_qb=1e-10):
    nA = np.linalg.norm(A)
    Qg = g["Q"].cpu().numpy()
    Bg = g["B"].cpu().numpy()
    if not in_tie_zone(o, eps):
        assert g["k"] == o.k, (g["k"], o.k)
        assert g["status"] == o.status
    k = g["k"]
    if k > 0:
        assert np.abs(Qg.T @ Qg - np.eye(k)).max() <= tol_orth
    if g["k"] == o.k and k > 0:
        diff = np.hstack([Qg, o.Q]) @ np.vstack([Bg, -o.B])
        assert np.linalg.norm(diff) / nA <= tol_qb
    true = np.linalg.norm(A - Qg @ Bg)
    if g["status"] == 0:
        assert true <= eps * (1 + 1e-8)
    # direct residual reported by the library = true residual of the returned factors
    assert abs(g["resid"] - true) <= 1e-12 * nA + 1e-8 * true
    return true


# ------------------------------------------------------------------------- Ω generator
@pytest.mark.parametrize("seed,n,row0,row1,col0,w", [
    (1, 300, 0, 300, 0, 10), (1, 1001, 0, 1001, 37, 64), (7, 1001, 1, 1000, 3, 5),
    (123456789012345, 50_001, 17, 49_999, 1000, 3), (2**64 - 1, 64, 0, 64, 2**33, 2)])
def test_omega_bitwise(qbmod, ctx, seed, n, row0, row1, col0, w):
    ldo = w + 3
    out = torch.full((row1 - row0, ldo), float("nan"), dtype=torch.float64, device="cuda")
    qbmod.qb_omega(ctx.ctx, seed, row0, row1, col0, w, out.data_ptr(), ldo)
    torch.cuda.synchronize()
    got = out[:, :w].cpu().numpy()
    ref = oomega.omega_panel(seed, n, col0, w, row0, row1)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    assert np.isnan(out[:, w:].cpu().numpy()).all()  # ldo padding untouched


# ------------------------------------------------------------------------- orth
@pytest.mark.parametrize("m,w", [(1000, 1), (1000, 7), (333, 64), (5000, 256), (2048, 128), (3000, 97), (3000, 100),
                                 (3000, 130), (3000, 200), (3000, 250)])
def test_orth_parity(qbmod, ctx, m, w):
    X = np.random.default_rng(m + w).standard_normal((m, w))
    Xd = to_dev(X)
    qbmod.qb_orth(ctx.ctx, Xd.data_ptr(), m, w, m)
    Q = Xd.cpu().numpy()
    Qo = oqb.orth(X)
    assert np.abs(Q.T @ Q - np.eye(w)).max() <= 1e-13
    assert np.abs(Q - Qo).max() <= 1e-11


def test_orth_rank_deficient_fallback(qbmod, ctx):
    rng = np.random.default_rng(4)
    X = rng.standard_normal((500, 12)) @ rng.standard_normal((12, 20))   # rank 12 < w = 20
    Xd = to_dev(X)
    qbmod.qb_orth(ctx.ctx, Xd.data_ptr(), 500, 20, 500)
    Q = Xd.cpu().numpy()
    assert np.abs(Q.T @ Q - np.eye(20)).max() <= 1e-12
    assert np.linalg.norm(X - Q @ (Q.T @ X)) <= 1e-12 * np.linalg.norm(X)


# ------------------------------------------------------------------------- full loop
CASES = [
    # name, m, n, spectrum, eps, b, q
    ("C1", 400, 300, "exp10_20", 1e-6, 10, 0),
    ("C1q1", 400, 300, "exp10_20", 1e-6, 10, 1),
    ("ragged", 333, 517, "exp10_25", 1e-7, 17, 0),
    ("tall_q2", 1000, 260, "poly2", 1e-5, 64, 2),
    ("wide", 260, 1000, "exp_100", 1e-4, 32, 1),
    ("b1", 120, 90, "exp10_20", 1e-3, 1, 0),
    ("bigb", 700, 650, "exp10_25", 1e-6, 256, 0),
]


def make(m, n, kind, seed):
    r = min(m, n)
    if kind == "exp10_25":
        sig = 10.0 ** (-np.arange(1, r + 1) / 25.0)
    else:
        sig = synth.sigma(kind, r)
    return synth.make_matrix_np(m, n, sig, seed), sig


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_factor_parity(qbmod, ctx, case):
    name, m, n, kind, eps, b, q = case
    A, sig = make(m, n, kind, 1000 + m)
    o = oqb.randqb_pb(A, eps, b, q, seed=1)
    g = ctx.factor(to_dev(A), eps, b, q, seed=1)
    check_parity(A, g, o, eps)
    # per-block residual history and the error indicator
    assert len(g["stats"]) == len(o.hist)
    nA2 = np.linalg.norm(A) ** 2
    for sg, ho in zip(g["stats"], o.hist):
        assert sg["ell"] == ho[0] and sg["w"] == ho[1]
        assert abs(sg["r2"] - ho[2]) <= 1e-12 * nA2
        assert abs(sg["ei"] - sg["r2"]) <= 6 * 2.0 ** -53 * nA2   # reading R1: 6 u ||A||^2


def test_config_C2_parity(qbmod, ctx):
    cfg = synth.CONFIGS["C2"]
    sig = synth.config_sigma(cfg)
    Ad = synth.make_matrix_torch(cfg.m, cfg.n, sig, cfg.seed_matrix)
    A = Ad.cpu().numpy()
    o = oqb.randqb_pb(A, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega)
    g = ctx.factor(Ad, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega)
    check_parity(A, g, o, cfg.eps)
    assert g["k"] >= synth.eps_rank(sig, cfg.eps)


def test_degenerate_inputs(qbmod, ctx):
    A = np.zeros((50, 40))
    g = ctx.factor(to_dev(A), 1e-8, 8)
    assert (g["status"], g["k"]) == (0, 0)
    A = np.random.default_rng(0).standard_normal((50, 40))
    g = ctx.factor(to_dev(A), 10 * np.linalg.norm(A), 8)       # reading R3
    assert (g["status"], g["k"]) == (0, 0)
    g = ctx.factor(to_dev(A), 0.0, 8, kmax=20)                 # reading R5
    assert (g["status"], g["k"]) == (qbmod.QB_NOT_CONVERGED, 20)
    assert [s["w"] for s in g["stats"]] == [8, 8, 4]
    o = oqb.randqb_pb(A, 0.0, 8, kmax=20)
    check_parity(A, g, o, 0.0)
    g = ctx.factor(to_dev(A), 1e-9, 8)                         # exhausts at min(m, n)
    assert g["k"] == 40 and g["resid"] < 1e-9


def test_empty_inputs(qbmod, ctx):
    """m = 0 or n = 0: k = 0 like the oracle (reading R3); b, q, eps are still validated, and
    rqb_svd / qb_pivoted_qr of the empty factorization return empty factors."""
    for shape in ((0, 7), (7, 0), (0, 0)):
        A = torch.zeros(shape, dtype=torch.float64, device="cuda")
        o = oqb.randqb_pb(np.zeros(shape), 0.0, 4)
        g = ctx.factor(A, 0.0, 4)
        assert (g["status"], g["k"]) == (o.status, o.k) == (0, 0)
        assert tuple(g["Q"].shape) == (shape[0], 0) and tuple(g["B"].shape) == (0, shape[1])
        assert g["resid"] == 0.0
        sv = ctx.svd()
        assert tuple(sv["U"].shape) == (shape[0], 0) and tuple(sv["V"].shape) == (shape[1], 0)
        pq = ctx.pivoted_qr()
        assert list(pq["perm"]) == list(range(shape[1])) and tuple(pq["R"].shape) == (0, shape[1])
        with pytest.raises(qbmod.QBError):
            ctx.factor(A, 1e-3, 0)
        with pytest.raises(qbmod.QBError):
            ctx.factor(A, -1.0, 4)


def test_rank_exhaustion_inside_block(qbmod, ctx):
    rng = np.random.default_rng(2)
    A = rng.standard_normal((120, 25)) @ rng.standard_normal((25, 90))
    eps = 1e-9 * np.linalg.norm(A)
    g = ctx.factor(to_dev(A), eps, 10, q=0, seed=3)
    o = oqb.randqb_pb(A, eps, 10, q=0, seed=3)
    assert g["k"] == o.k == 30
    Qg = g["Q"].cpu().numpy()
    assert np.abs(Qg.T @ Qg - np.eye(30)).max() <= 1e-12
    assert np.linalg.norm(A - Qg @ g["B"].cpu().numpy()) <= 1e-12 * np.linalg.norm(A)
    assert sum(s["fallback"] for s in g["stats"]) >= 1


def test_invalid_arguments(qbmod, ctx):
    A = to_dev(np.ones((10, 10)))
    with pytest.raises(qbmod.QBError):
        ctx.factor(A, 1e-3, 0)
    with pytest.raises(qbmod.QBError):
        ctx.factor(A, -1.0, 4)
    An = np.ones((10, 10))
    An[3, 4] = np.nan
    with pytest.raises(qbmod.QBError) as e:
        ctx.factor(to_dev(An), 1e-3, 4)
    assert e.value.status == qbmod.QB_ERR_INVALID_ARG


def test_overwrite_a_leaves_residual(qbmod, ctx):
    A, _ = make(300, 200, "exp10_25", 5)
    Ad = to_dev(A)
    g = ctx.factor(Ad, 1e-6, 16, overwrite=True)
    R = Ad.cpu().numpy()
    Qg, Bg = g["Q"].cpu().numpy(), g["B"].cpu().numpy()
    assert np.linalg.norm(R - (A - Qg @ Bg)) <= 1e-12 * np.linalg.norm(A)
    g2 = ctx.factor(to_dev(A), 1e-6, 16)
    assert g2["k"] == g["k"]
    assert np.array_equal(g2["Q"].cpu().numpy(), Qg)   # bitwise reproducible


def test_no_reproj_loses_orthogonality(qbmod, ctx):
    """without line (3') the blocks drift into the earlier span."""
    A, _ = make(1000, 800, "exp10_25", 3)
    g = ctx.factor(to_dev(A), 1e-13, 20, q=0, seed=1)
    r = qbmod.qb_factor(ctx.ctx, to_dev(A).data_ptr(), 1000, 800, 1000, 1e-13, 20, 0, 1, 0, qbmod.QB_NO_REPROJ)
    Q = g["Q"].cpu().numpy()
    Qn = qbmod.view_colmajor(r["Q"], 1000, r["k"], r["ldq"]).cpu().numpy()
    o_with = np.abs(Q.T @ Q - np.eye(Q.shape[1])).max()
    o_without = np.abs(Qn.T @ Qn - np.eye(Qn.shape[1])).max()
    assert o_with <= 1e-12 and o_without > 1e3 * o_with


def test_target_config_properties(qbmod, ctx):
    """The bench workload (T: 20000^2, b = 256, q = 0) at full size, in the launch configuration
    bench.py times: properties that hold at any size + sampled Ω entries vs the oracle."""
    cfg = synth.CONFIGS["T"]
    sig = synth.config_sigma(cfg)
    Ad = synth.make_matrix_torch(cfg.m, cfg.n, sig, cfg.seed_matrix)
    nA = float(torch.linalg.norm(Ad))
    g = ctx.factor(Ad, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega, copy_out=False)
    Q, B, k = g["Q"], g["B"], g["k"]
    assert g["status"] == 0 and k % cfg.b == 0
    kq = synth.eps_rank(sig, cfg.eps)
    assert k >= kq
    orth = (Q.T @ Q - torch.eye(k, dtype=torch.float64, device="cuda")).abs().max().item()
    assert orth <= 1e-12
    true = torch.linalg.norm(torch.addmm(Ad, Q, B, alpha=-1.0)).item()
    assert true <= cfg.eps * (1 + 1e-8)
    assert true >= synth.optimal_error(sig, k) * (1 - 1e-6)
    st = g["stats"]
    assert st[-1]["r2"] <= cfg.eps ** 2 < st[-2]["r2"]
    for s in st:
        assert abs(s["ei"] - s["r2"]) <= 6 * 2.0 ** -53 * nA ** 2   # reading R1: 6 u ||A||^2
    # sampled Ω(rows, cols) at the full size against the oracle generator
    rng = np.random.default_rng(0)
    for c0 in (0, k - cfg.b):
        rows = rng.integers(0, cfg.n, 64)
        out = torch.empty((cfg.n, cfg.b), dtype=torch.float64, device="cuda")
        qbmod.qb_omega(ctx.ctx, cfg.seed_omega, 0, cfg.n, c0, cfg.b, out.data_ptr(), cfg.b)
        got = out.cpu().numpy()[rows]
        ref = np.vstack([oomega.omega_panel(cfg.seed_omega, cfg.n, c0, cfg.b, r, r + 1) for r in rows])
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


def test_c4_config_properties_fp32(qbmod):
    """BASELINE configs[3] (C4: 200000 x 2000 FP32, b = 128) at full size on the FP32 tensor-core
    path: properties that hold at any size, at the north_star's FP32 tolerances."""
    cfg = synth.CONFIGS["C4"]
    sig = synth.config_sigma(cfg)
    A32 = synth.make_matrix_torch(cfg.m, cfg.n, sig, cfg.seed_matrix, dtype=torch.float32)
    c = qbmod.QB(0, dtype=qbmod.QB_F32)
    g = c.factor(A32, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega, copy_out=True)
    c.close()
    k = g["k"]
    assert g["status"] == 0 and k % cfg.b == 0 and k >= synth.eps_rank(sig, cfg.eps)
    Q, B = g["Q"].double(), g["B"].double()
    A = A32.double()
    nA = float(torch.linalg.norm(A))
    orth = (Q.T @ Q - torch.eye(k, dtype=torch.float64, device="cuda")).abs().max().item()
    assert orth <= 1e-5
    true = torch.linalg.norm(torch.addmm(A, Q, B, alpha=-1.0)).item()
    assert true <= cfg.eps * (1 + 1e-4) + 1e-6 * nA
    assert abs(g["resid"] - true) <= 1e-6 * nA
    assert true >= synth.optimal_error(sig, k) * (1 - 1e-3)
    st = g["stats"]
    assert st[-1]["r2"] <= cfg.eps ** 2 < st[-2]["r2"]


def test_fresh_context_reproducible_across_growth(qbmod):
    """k > 1024 forces the Q̄/B̄ capacity to grow inside the first call; a fresh context and a
    reused one must give bitwise identical factors (fixed-order reductions)."""
    sig = np.exp(-np.arange(1, 3001) / 100.0)
    Ad = synth.make_matrix_torch(3000, 3000, sig, 77)
    c = qbmod.QB(0)
    g1 = c.factor(Ad, 1e-4, 64, 0, seed=5)
    g2 = c.factor(Ad, 1e-4, 64, 0, seed=5)
    c.close()
    assert g1["k"] == g2["k"] and g1["k"] > 1024
    assert torch.equal(g1["Q"], g2["Q"]) and torch.equal(g1["B"], g2["B"])
    assert [s["r2"] for s in g1["stats"]] == [s["r2"] for s in g2["stats"]]


@pytest.mark.parametrize("q", [0, 1])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_distributed_context_single_rank_bitwise(qbmod, q, dt):
    """A column-sharded context (NCCL communicator of one rank) runs the allreduce code path
    and must reproduce the plain context bit for bit.  FP32: the plain context takes Y's FP32
    copy from the sketch's epilogue, the sharded one converts the all-reduced Y; same values."""
    try:
        uid = qbmod.qb_nccl_unique_id()
    except qbmod.QBError:
        pytest.skip("NCCL not loadable")
    A, _ = make(600, 500, "exp10_25", 9)
    f32 = dt == "f32"
    dtype = qbmod.QB_F32 if f32 else qbmod.QB_F64
    Ad = torch.from_numpy(np.asfortranarray(A.astype(np.float32))).cuda() if f32 else to_dev(A)
    eps = 1e-4 if f32 else 1e-8
    plain = qbmod.QB(0, dtype=dtype)
    g0 = plain.factor(Ad.clone(), eps, 32, q, seed=4)
    plain.close()
    d = qbmod.QB(0, dtype=dtype, dist=dict(rank=0, nranks=1, unique_id=uid, col_offset=0, n_global=500))
    g1 = d.factor(Ad.clone(), eps, 32, q, seed=4)
    d.close()
    assert g0["k"] == g1["k"]
    assert torch.equal(g0["Q"], g1["Q"]) and torch.equal(g0["B"], g1["B"])


@pytest.mark.parametrize("q", [0, 1])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_row_sharded_context_single_rank(qbmod, q, dt):
    """A row-sharded context (NEXT-2; NCCL communicator of one rank) runs the Gram / W / Z / B_i
    allreduce code path; against the oracle like a plain context (FP32: FP32 tolerances)."""
    try:
        uid = qbmod.qb_nccl_unique_id()
    except qbmod.QBError:
        pytest.skip("NCCL not loadable")
    A, _ = make(3000, 200, "exp_100", 19)
    eps = 1e-3 if dt == "f32" else 1e-8
    d = qbmod.QB(0, dtype=qbmod.QB_F32 if dt == "f32" else qbmod.QB_F64,
                 dist=dict(shard="rows", rank=0, nranks=1, unique_id=uid, row_offset=0, m_global=3000))
    if dt == "f32":
        A32 = A.astype(np.float32)
        Aw = A32.astype(np.float64)
        o = oqb.randqb_pb(Aw, eps, 32, q, seed=4, omega_dtype=np.float32)
        g = d.factor(torch.from_numpy(np.asfortranarray(A32)).cuda(), eps, 32, q, seed=4)
        assert g["k"] == o.k
        Qg, Bg = g["Q"].double().cpu().numpy(), g["B"].double().cpu().numpy()
        nA = np.linalg.norm(Aw)
        assert np.abs(Qg.T @ Qg - np.eye(g["k"])).max() <= 1e-5
        assert np.linalg.norm(np.hstack([Qg, o.Q]) @ np.vstack([Bg, -o.B])) / nA <= 1e-4
        assert np.linalg.norm(Aw - Qg @ Bg) <= eps * (1 + 1e-4) + 1e-6 * nA
    else:
        o = oqb.randqb_pb(A, eps, 32, q, seed=4)
        g = d.factor(to_dev(A), eps, 32, q, seed=4)
        check_parity(A, g, o, eps)
        s = d.svd()   # rqb_svd on a row-sharded context (B replicated)
        np.testing.assert_allclose(s["S"].cpu().numpy(), np.linalg.svd(o.B, compute_uv=False),
                                   rtol=0, atol=1e-10 * np.linalg.norm(A))
    d.close()


@pytest.mark.parametrize("case", [(400, 300, "exp10_20", 1e-4, 10, 0), (3000, 200, "exp_100", 1e-3, 32, 0),
                                  (1000, 260, "poly2", 1e-4, 64, 1), (5000, 700, "exp_100", 1e-3, 100, 0),
                                  (2000, 1500, "exp_150", 1e-3, 256, 0), (3000, 500, "exp_100", 1e-3, 96, 2)])
def test_fp32_path_parity(qbmod, case):
    """FP32 path (BASELINE configs[3] family): float A in, float Q, B out, ragged block widths
    (b = 10, 96, 100) and b = 256 through the 3xTF32 GEMMs, q = 0..2.  The oracle runs in
    FP64 on the same FP32 input with Ω = RN_32(Ω) (reading R18); north_star FP32 tolerances
    1e-5 (orthogonality) and 1e-4 (QB parity)."""
    m, n, kind, eps, b, q = case
    A64, _ = make(m, n, kind, 31 + m)
    A32 = A64.astype(np.float32)
    Aw = A32.astype(np.float64)
    o = oqb.randqb_pb(Aw, eps, b, q, seed=2, omega_dtype=np.float32)
    c = qbmod.QB(0, dtype=qbmod.QB_F32)
    g = c.factor(torch.from_numpy(np.asfortranarray(A32)).cuda(), eps, b, q, seed=2)
    c.close()
    assert g["Q"].dtype == torch.float32 and g["B"].dtype == torch.float32
    assert g["k"] == o.k
    Qg = g["Q"].double().cpu().numpy()
    Bg = g["B"].double().cpu().numpy()
    nA = np.linalg.norm(Aw)
    assert np.abs(Qg.T @ Qg - np.eye(g["k"])).max() <= 1e-5
    assert np.linalg.norm(np.hstack([Qg, o.Q]) @ np.vstack([Bg, -o.B])) / nA <= 1e-4
    assert np.linalg.norm(Aw - Qg @ Bg) <= eps * (1 + 1e-4) + 1e-6 * nA


@pytest.mark.parametrize("q", [1, 2])
def test_skip_power_orth_parity(qbmod, ctx, q):
    """NEXT-3: the blocked scheme without re-orthonormalisation between
    applications of A and A^* (flag QB_SKIP_POWER_ORTH) against the oracle's same variant."""
    A, _ = make(600, 400, "exp10_25", 3)
    eps = 1e-7
    o = oqb.randqb_pb(A, eps, 20, q, seed=1, skip_power_orth=True)
    g = ctx.factor(to_dev(A), eps, 20, q, seed=1, flags=qbmod.QB_SKIP_POWER_ORTH)
    check_parity(A, g, o, eps)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_factor_host_entry_point(qbmod, dt):
    """qb_factor_host (the end-to-end entry point): host A in, Q / B streamed to host buffers block
    by block (overlapping the next block); equal to the device entry point's factors, and kcap
    truncates the copy."""
    A, _ = make(900, 700, "exp10_25", 23)
    npdt = np.float32 if dt == "f32" else np.float64
    Ah = np.asfortranarray(A.astype(npdt))
    c = qbmod.QB(0, dtype=qbmod.QB_F32 if dt == "f32" else qbmod.QB_F64)
    g = c.factor(torch.from_numpy(Ah).cuda(), 1e-5, 32, 0, seed=3)
    k = g["k"]
    for kcap in (k + 5, k - 40):
        Qh = np.full((kcap, 900), np.nan, dtype=npdt)      # column-major 900 x kcap
        Bh = np.full((kcap, 700), np.nan, dtype=npdt)      # row-major kcap x 700
        r = qbmod.qb_factor_host(c.ctx, Ah.ctypes.data, 900, 700, 900, 1e-5, 32, 0, 3, 0, Qh.ctypes.data, 900,
                                 Bh.ctypes.data, 700, kcap)
        assert r["k"] == k and abs(r["resid"] - g["resid"]) <= 1e-12 * np.linalg.norm(A)
        kc = min(k, kcap)
        assert np.array_equal(Qh[:kc].T, g["Q"][:, :kc].cpu().numpy())
        assert np.array_equal(Bh[:kc], g["B"][:kc].cpu().numpy())
        assert np.isnan(Qh[kc:]).all() and np.isnan(Bh[kc:]).all()
    c.close()


def test_factor_host_kmax_reached(qbmod):
    """qb_factor_host when kmax ends the loop before the stop test fires (QB_NOT_CONVERGED): the last
    block's host copy is still issued, and the host factors equal the device entry point's."""
    A, _ = make(900, 700, "exp10_25", 23)
    Ah = np.asfortranarray(A)
    c = qbmod.QB(0)
    g = c.factor(torch.from_numpy(Ah).cuda(), 1e-12, 32, 0, seed=3, kmax=96)
    assert g["status"] == qbmod.QB_NOT_CONVERGED and g["k"] == 96
    Qh = np.full((96, 900), np.nan)
    Bh = np.full((96, 700), np.nan)
    r = qbmod.qb_factor_host(c.ctx, Ah.ctypes.data, 900, 700, 900, 1e-12, 32, 0, 3, 96, Qh.ctypes.data, 900,
                             Bh.ctypes.data, 700, 96)
    assert r["status"] == qbmod.QB_NOT_CONVERGED and r["k"] == 96
    assert np.array_equal(Qh.T, g["Q"].cpu().numpy())
    assert np.array_equal(Bh, g["B"].cpu().numpy())
    c.close()


def test_orth_fp32_context(qbmod):
    """qb_orth on an FP32 context: FP64 CholeskyQR2 of the widened panel, rounded to FP32."""
    X = np.random.default_rng(4).standard_normal((3000, 100)).astype(np.float32)
    Xd = torch.from_numpy(np.asfortranarray(X)).cuda()
    c = qbmod.QB(0, dtype=qbmod.QB_F32)
    qbmod.qb_orth(c.ctx, Xd.data_ptr(), 3000, 100, 3000)
    c.close()
    Q = Xd.double().cpu().numpy()
    Qo = oqb.orth(X.astype(np.float64))
    assert np.abs(Q.T @ Q - np.eye(100)).max() <= 1e-6
    assert np.abs(Q - Qo).max() <= 1e-6


@pytest.mark.parametrize("case", [("C1", 400, 300, "exp10_20", 1e-6, 10, 0), ("C1q1", 400, 300, "exp10_20", 1e-6, 10, 1),
                                  ("ragged", 333, 517, "exp10_25", 1e-7, 17, 0), ("q2", 300, 200, "poly2", 1e-5, 24, 2),
                                  ("b64", 500, 400, "exp10_25", 1e-8, 64, 0), ("b1", 120, 90, "exp10_20", 1e-3, 1, 0)],
                         ids=lambda c: c[0])
def test_small_loop_matches_general_path_and_oracle(qbmod, ctx, case):
    """The one-launch cluster path (small_loop.cuh) for problems that fit in shared memory runs the
    same loop as the general path: both against the oracle (k, products, per-block r^2) and
    against each other (QB_FORCE_GENERAL)."""
    name, m, n, kind, eps, b, q = case
    A, _ = make(m, n, kind, 2000 + m)
    o = oqb.randqb_pb(A, eps, b, q, seed=7)
    g_small = ctx.factor(to_dev(A), eps, b, q, seed=7)
    g_gen = ctx.factor(to_dev(A), eps, b, q, seed=7, flags=qbmod.QB_FORCE_GENERAL)
    nA2 = np.linalg.norm(A) ** 2
    for g in (g_small, g_gen):
        check_parity(A, g, o, eps)
        assert len(g["stats"]) == len(o.hist)
        for sg, ho in zip(g["stats"], o.hist):
            assert sg["ell"] == ho[0] and sg["w"] == ho[1]
            assert abs(sg["r2"] - ho[2]) <= 1e-12 * nA2
            assert abs(sg["ei"] - sg["r2"]) <= 6 * 2.0 ** -53 * nA2
    d = np.hstack([g_small["Q"].cpu().numpy(), g_gen["Q"].cpu().numpy()]) @ \
        np.vstack([g_small["B"].cpu().numpy(), -g_gen["B"].cpu().numpy()])
    assert np.linalg.norm(d) <= 1e-12 * np.sqrt(nA2)
    # bitwise reproducible from call to call
    g2 = ctx.factor(to_dev(A), eps, b, q, seed=7)
    assert torch.equal(g2["Q"], g_small["Q"]) and torch.equal(g2["B"], g_small["B"])


def test_small_loop_overwrite_and_host_entry(qbmod, ctx):
    """QB_OVERWRITE_A leaves the residual in A; qb_factor_host returns the same factors."""
    A, _ = make(300, 200, "exp10_25", 5)
    Ad = to_dev(A)
    g = ctx.factor(Ad, 1e-6, 16, overwrite=True)
    Qg, Bg = g["Q"].cpu().numpy(), g["B"].cpu().numpy()
    assert np.linalg.norm(Ad.cpu().numpy() - (A - Qg @ Bg)) <= 1e-12 * np.linalg.norm(A)
    Ah = np.asfortranarray(A)
    k = g["k"]
    Qh = np.full((k, 300), np.nan)
    Bh = np.full((k, 200), np.nan)
    r = qbmod.qb_factor_host(ctx.ctx, Ah.ctypes.data, 300, 200, 300, 1e-6, 16, 0, 1, 0, Qh.ctypes.data, 300,
                             Bh.ctypes.data, 200, k)
    assert r["k"] == k
    assert np.array_equal(Qh.T, Qg) and np.array_equal(Bh, Bg)


@pytest.mark.parametrize("force_general", [False, True])
def test_kappa_proxy_matches_oracle_sketch(qbmod, ctx, force_general):
    """qb_stats' kappa-proxy: max R_jj / min R_jj of the block's first CholeskyQR
    factorization, i.e. of the sketch Y_i = A^(i-1) Omega_i, equals the ratio of |diag R| of the
    economy QR of the oracle's Y_i (the R of a full-rank QR is unique up to row signs)."""
    A, _ = make(400, 300, "exp10_20", 1400)
    eps, b = 1e-6, 10
    o = oqb.randqb_pb(A, eps, b, 0, seed=1)
    g = ctx.factor(to_dev(A), eps, b, 0, seed=1, flags=qbmod.QB_FORCE_GENERAL if force_general else 0)
    assert g["k"] == o.k
    for i, st in enumerate(g["stats"]):
        ell = i * b
        R = A - o.Q[:, :ell] @ o.B[:ell]                      # A^(i-1) from the oracle's factors
        Y = R @ oqb.omega(1, A.shape[1], ell, b)
        d = np.abs(np.diag(np.linalg.qr(Y, mode="r")))
        assert st["kappa_r"] > 1.0
        assert abs(st["kappa_r"] - d.max() / d.min()) <= 1e-6 * d.max() / d.min(), (i, st["kappa_r"], d.max() / d.min())
