"""The library's SHARDED code path with P = 2 and 4 ranks on one GPU.

Each rank is a context of its own (qb_create_sharded with an in-process loopback group, one host
thread and one stream per rank) holding its column shard (square A) or row shard (tall-skinny A,
NEXT-2).  The exchange steps — the Y_i sums, the power step's Gram, the re-projection W, B_i and
the norm scalars — run through the loopback collective: every rank's stream is finished on the
host, then one kernel sums all ranks' buffers in rank order (no kernel waits on another rank).
Everything else is the exact library code that runs under NCCL on P GPUs.

The sharded factorization is compared with the UNSHARDED oracle on the same A and seed
(north_star tolerances, reading R19 for k): identical k, ||Q^T Q - I||_max, product parity
[Q_g Q_o][B_g; -B_o] and the per-block residual r_i^2 — the paper's loop (Fig. 2 / Fig. 4,
PAPER.md:698-725, :859-887) is the same for every P because Ω is indexed by global row and
column (reading R15)."""
import threading

import numpy as np
import pytest

import synth
from oracle import qb as oqb
from paper_1503_07157_b200.dist import shard_columns

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def qbmod():
    import paper_1503_07157_b200 as qbp
    from paper_1503_07157_b200 import build
    build.build()
    return qbp


def make(m, n, kind, seed):
    r = min(m, n)
    sig = 10.0 ** (-np.arange(1, r + 1) / 25.0) if kind == "exp10_25" else synth.sigma(kind, r)
    return synth.make_matrix_np(m, n, sig, seed)


def run_loopback(qbmod, A, P, shard, eps, b, q, seed, f32=False, bad_rank=None, flags=0):
    """Factor A on P in-process ranks.  Returns the per-rank result dicts (or exceptions)."""
    import ctypes
    m, n = A.shape
    grp = qbmod.qb_loopback_create(P)
    npdt = np.float32 if f32 else np.float64
    ctxs, streams, parts = [], [], []
    for r in range(P):
        off, cnt = shard_columns(n if shard == "cols" else m, P, r)
        Ar = A[:, off:off + cnt] if shard == "cols" else A[off:off + cnt, :]
        parts.append(torch.from_numpy(np.asfortranarray(Ar.astype(npdt))).cuda())
        st = torch.cuda.Stream()
        streams.append(st)
        d = dict(loopback=grp, rank=r, nranks=P)
        if shard == "cols":
            d.update(col_offset=off, n_global=n)
        else:
            d.update(shard="rows", row_offset=off, m_global=m)
        ctxs.append(qbmod.QB(0, dtype=qbmod.QB_F32 if f32 else qbmod.QB_F64,
                             stream=ctypes.c_void_p(st.cuda_stream), dist=d))
    torch.cuda.synchronize()
    out = [None] * P

    def work(r):
        try:
            with torch.cuda.stream(streams[r]):
                out[r] = ctxs[r].factor(parts[r], eps, 0 if r == bad_rank else b, q, seed=seed, flags=flags)
                streams[r].synchronize()
        except Exception as e:  # noqa: BLE001 - reported per rank
            out[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a loopback rank hung"
    for c in ctxs:
        c.close()
    qbmod.qb_loopback_destroy(grp)
    return out


def assemble(out, shard):
    """Global Q, B from the shards: column shards replicate Q (bitwise on every rank) and split
    B by columns; row shards split Q by rows and replicate B."""
    for g in out:
        assert not isinstance(g, Exception), g
    ks = {g["k"] for g in out}
    assert len(ks) == 1, ks
    if shard == "cols":
        for g in out[1:]:
            assert torch.equal(g["Q"], out[0]["Q"])       # the replicated orth is bitwise identical
        Q = out[0]["Q"].double().cpu().numpy()
        B = np.hstack([g["B"].double().cpu().numpy() for g in out])
    else:
        for g in out[1:]:
            assert torch.equal(g["B"], out[0]["B"])
        Q = np.vstack([g["Q"].double().cpu().numpy() for g in out])
        B = out[0]["B"].double().cpu().numpy()
    for g in out[1:]:
        assert [s["r2"] for s in g["stats"]] == [s["r2"] for s in out[0]["stats"]]
    return ks.pop(), Q, B, out[0]["stats"], out[0]["resid"]


def check_vs_oracle(A, o, k, Q, B, stats, resid, eps, f32):
    tol_orth, tol_qb, tol_r2 = (1e-5, 1e-4, 1e-6) if f32 else (1e-12, 1e-10, 1e-12)
    nA = np.linalg.norm(A)
    assert k == o.k
    assert np.abs(Q.T @ Q - np.eye(k)).max() <= tol_orth
    assert np.linalg.norm(np.hstack([Q, o.Q]) @ np.vstack([B, -o.B])) / nA <= tol_qb
    assert len(stats) == len(o.hist)
    for s, h in zip(stats, o.hist):
        assert s["ell"] == h[0] and s["w"] == h[1]
        assert abs(s["r2"] - h[2]) <= tol_r2 * nA ** 2
    true = np.linalg.norm(A - Q @ B)
    assert true <= eps * (1 + (1e-4 if f32 else 1e-8)) + (1e-6 * nA if f32 else 0.0)
    assert abs(resid - true) <= (1e-6 if f32 else 1e-12) * nA + 1e-8 * true


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("q", [0, 1])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_column_shards_match_unsharded_oracle(qbmod, P, q, dt):
    """Square A split by columns (ragged: 1001 columns over P ranks, odd offsets split Ω's row
    pairs), Y_i / power-step Gram / scalars summed across the ranks."""
    f32 = dt == "f32"
    A = make(900, 1001, "exp10_25", 41)
    eps = 1e-4 if f32 else 1e-8
    Aw = A.astype(np.float32).astype(np.float64) if f32 else A
    o = oqb.randqb_pb(Aw, eps, 32, q, seed=5, omega_dtype=np.float32 if f32 else np.float64)
    out = run_loopback(qbmod, A, P, "cols", eps, 32, q, 5, f32=f32)
    k, Q, B, stats, resid = assemble(out, "cols")
    check_vs_oracle(Aw, o, k, Q, B, stats, resid, eps, f32)


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("q", [0, 1])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_row_shards_match_unsharded_oracle(qbmod, P, q, dt):
    """Tall-skinny A (C4-shaped, 20000 x 300) split by rows (NEXT-2): Grams, W, Z and B_i summed
    across the ranks, Q row-distributed, B replicated."""
    f32 = dt == "f32"
    A = make(20000, 300, "exp_100", 43)
    eps = 1e-3 if f32 else 1e-8
    Aw = A.astype(np.float32).astype(np.float64) if f32 else A
    o = oqb.randqb_pb(Aw, eps, 32, q, seed=6, omega_dtype=np.float32 if f32 else np.float64)
    out = run_loopback(qbmod, A, P, "rows", eps, 32, q, 6, f32=f32)
    k, Q, B, stats, resid = assemble(out, "rows")
    check_vs_oracle(Aw, o, k, Q, B, stats, resid, eps, f32)


def test_column_shards_b256_reprojection(qbmod):
    """b = 256 (the target's block size) over 2 column shards, several blocks with re-projection."""
    A = make(1500, 1400, "exp_150", 47)
    o = oqb.randqb_pb(A, 1e-3, 256, 0, seed=2)
    out = run_loopback(qbmod, A, 2, "cols", 1e-3, 256, 0, 2)
    k, Q, B, stats, resid = assemble(out, "cols")
    assert len(stats) >= 3
    check_vs_oracle(A, o, k, Q, B, stats, resid, 1e-3, False)


def test_skip_power_orth_column_shards(qbmod):
    """NEXT-3 on column shards: Y = A (A^T Y) with the Z sums."""
    A = make(700, 640, "exp10_25", 53)
    o = oqb.randqb_pb(A, 1e-7, 20, 1, seed=1, skip_power_orth=True)
    out = run_loopback(qbmod, A, 2, "cols", 1e-7, 20, 1, 1, flags=qbmod.QB_SKIP_POWER_ORTH)
    k, Q, B, stats, resid = assemble(out, "cols")
    check_vs_oracle(A, o, k, Q, B, stats, resid, 1e-7, False)


def test_failing_rank_releases_its_peers(qbmod):
    """A rank that fails (here: b = 0, rejected before its first collective) aborts the group:
    its peers return QB_ERR_NCCL from the next collective instead of waiting forever."""
    A = make(300, 400, "exp10_25", 59)
    out = run_loopback(qbmod, A, 3, "cols", 1e-6, 16, 0, 1, bad_rank=1)
    assert isinstance(out[1], qbmod.QBError) and out[1].status == qbmod.QB_ERR_INVALID_ARG
    for r in (0, 2):
        assert isinstance(out[r], qbmod.QBError) and out[r].status == qbmod.QB_ERR_NCCL


def test_loopback_group_validation(qbmod):
    with pytest.raises(qbmod.QBError):
        qbmod.qb_loopback_create(0)
    with pytest.raises(qbmod.QBError):
        qbmod.qb_loopback_create(qbmod.QB_LOOPBACK_MAX_RANKS + 1)
    g = qbmod.qb_loopback_create(2)
    with pytest.raises(qbmod.QBError):   # rank out of range
        qbmod.qb_create_sharded(0, 2, 2, qbmod.QB_SHARD_COLS, 0, 10, loopback=g)
    qbmod.qb_loopback_destroy(g)
