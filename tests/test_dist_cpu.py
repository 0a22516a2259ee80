"""The N > 1 (column- and row-sharded) paths on the CPU with torch.distributed gloo, world size 2.

The CUDA library shards A by columns: rank p owns A(:, off_p : off_p + n_p),
draws rows off_p.. of every Ω_i from global indices, and the only exchanges are sums — of
Y_i = Σ_p A_p Ω_p, of the power-step Gram Σ_p Z_pᵀ Z_p, and of the norm scalars.  These tests
check that decomposition against the unsharded oracle on real multi-process gloo collectives
(the same algebra the library performs with NCCL), plus the bootstrap: the column split and
the ncclUniqueId broadcast from rank 0.

Row sharding (NEXT-2, tall-skinny A): rank p owns A(off_p : off_p + m_p, :); Ω is replicated,
Y_i and Q_i stay local, and the sums are the CholeskyQR Grams Σ_p Y_pᵀY_p, the re-projection
W = Σ_p Q̄_pᵀQ_p, the power step's Z = Σ_p A_pᵀQ_p and B_i = Σ_p Q_pᵀA_p."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import omega as oomega
from oracle import qb as oqb
from paper_1503_07157_b200.dist import broadcast_unique_id, shard_columns, shard_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def sharded_randqb(A_p, off, n_global, eps, b, q, seed):
    """The library's column-sharded loop, written with oracle primitives and gloo sums."""
    m, n_p = A_p.shape
    R = A_p.copy()
    kmax = min(m, n_global)
    r2 = float(_allreduce(np.array([oqb.frob2(R)]))[0])
    if r2 <= eps * eps:
        return 0, np.zeros((m, 0)), np.zeros((0, n_p)), []
    Qs, Bs, hist, ell = [], [], [], 0
    while ell < kmax:
        w = min(b, kmax - ell)
        Om_p = oomega.omega_panel(seed, n_global, ell, w, off, off + n_p)   # this rank's rows of Ω_i
        Qi = oqb.orth(_allreduce(R @ Om_p))                                  # Y_i = Σ_p A_p Ω_p
        for _ in range(q):
            Z_p = R.T @ Qi                                                   # rows of Z live on their rank
            G = _allreduce(Z_p.T @ Z_p)                                      # distributed CholeskyQR
            Rz = np.linalg.cholesky(G).T
            Z_p = np.linalg.solve(Rz.T, Z_p.T).T
            Qi = oqb.orth(_allreduce(R @ Z_p))
        if ell > 0:
            Qbar = np.hstack(Qs)
            Qi = oqb.orth(Qi - Qbar @ (Qbar.T @ Qi))                        # replicated
        Bi = Qi.T @ R                                                        # local
        R = R - Qi @ Bi                                                      # local
        r2 = float(_allreduce(np.array([oqb.frob2(R)]))[0])
        Qs.append(Qi)
        Bs.append(Bi)
        ell += w
        hist.append((ell, r2))
        if r2 <= eps * eps:
            break
    return ell, np.hstack(Qs), np.vstack(Bs), hist


def _dist_orth(Y_p):
    """CholeskyQR2 of a row-distributed panel: Gram summed over the ranks, T applied locally."""
    for _ in range(2):
        G = _allreduce(Y_p.T @ Y_p)
        Rz = np.linalg.cholesky(G).T
        Y_p = np.linalg.solve(Rz.T, Y_p.T).T
    return Y_p


def sharded_rows_randqb(A_p, m_global, eps, b, q, seed):
    """The library's row-sharded loop (NEXT-2), written with oracle primitives and gloo sums."""
    m_p, n = A_p.shape
    R = A_p.copy()
    kmax = min(m_global, n)
    r2 = float(_allreduce(np.array([oqb.frob2(R)]))[0])
    if r2 <= eps * eps:
        return 0, np.zeros((m_p, 0)), np.zeros((0, n)), []
    Qs, Bs, hist, ell = [], [], [], 0
    while ell < kmax:
        w = min(b, kmax - ell)
        Om = oomega.omega_panel(seed, n, ell, w)                             # replicated Ω_i
        Qi = _dist_orth(R @ Om)                                              # Y_p local
        for _ in range(q):
            Z = oqb.orth(_allreduce(R.T @ Qi))                               # Z = Σ_p A_pᵀQ_p, replicated
            Qi = _dist_orth(R @ Z)
        if ell > 0:
            Qbar = np.hstack(Qs)
            Qi = _dist_orth(Qi - Qbar @ _allreduce(Qbar.T @ Qi))            # W = Σ_p Q̄_pᵀQ_p
        Bi = _allreduce(Qi.T @ R)                                            # B_i = Σ_p Q_pᵀA_p
        R = R - Qi @ Bi                                                      # local
        r2 = float(_allreduce(np.array([oqb.frob2(R)]))[0])
        Qs.append(Qi)
        Bs.append(Bi)
        ell += w
        hist.append((ell, r2))
        if r2 <= eps * eps:
            break
    return ell, np.hstack(Qs), np.vstack(Bs), hist


def _worker_rows(rank, world, port, q, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = synth.make_matrix_np(3000, 200, synth.sigma("exp_100", 200), 77)
        off, m_p = shard_rows(A.shape[0], world, rank)
        k, Q_p, B, hist = sharded_rows_randqb(A[off:off + m_p], A.shape[0], 1e-3, 32, q, 2)
        Qs = [None] * world
        dist.all_gather_object(Qs, Q_p)
        if rank == 0:
            out.put((k, np.vstack(Qs), B, hist))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q", [0, 1])
def test_row_sharded_loop_matches_oracle(q):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_rows, args=(r, 2, port, q, out)) for r in range(2)]
    for p in procs:
        p.start()
    k, Q, B, hist = out.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = synth.make_matrix_np(3000, 200, synth.sigma("exp_100", 200), 77)
    o = oqb.randqb_pb(A, 1e-3, 32, q, seed=2)
    assert k == o.k
    nA = np.linalg.norm(A)
    assert np.linalg.norm(np.hstack([Q, o.Q]) @ np.vstack([B, -o.B])) / nA <= 1e-10
    assert np.abs(Q.T @ Q - np.eye(k)).max() <= 1e-12
    for (ell, r2), ho in zip(hist, o.hist):
        assert ell == ho[0] and abs(r2 - ho[2]) <= 1e-12 * nA ** 2


def _worker(rank, world, port, q, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # bootstrap: rank 0's id reaches every rank
        uid = bytes(range(128)) if rank == 0 else bytes(128)
        got = broadcast_unique_id(uid)
        assert got == bytes(range(128))
        cfg = synth.CONFIGS["C1"]
        A = synth.make_matrix_np(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix)
        off, n_p = shard_columns(cfg.n, world, rank)
        k, Q, B_p, hist = sharded_randqb(A[:, off:off + n_p], off, cfg.n, cfg.eps, cfg.b, q, cfg.seed_omega)
        Bs = [None] * world
        dist.all_gather_object(Bs, B_p)
        if rank == 0:
            out.put((k, Q, np.hstack(Bs), hist))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q", [0, 1])
def test_column_sharded_loop_matches_oracle(q):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, out)) for r in range(2)]
    for p in procs:
        p.start()
    k, Q, B, hist = out.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synth.CONFIGS["C1"]
    A = synth.make_matrix_np(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix)
    o = oqb.randqb_pb(A, cfg.eps, cfg.b, q, seed=cfg.seed_omega)
    assert k == o.k
    nA = np.linalg.norm(A)
    assert np.linalg.norm(np.hstack([Q, o.Q]) @ np.vstack([B, -o.B])) / nA <= 1e-10
    assert np.abs(Q.T @ Q - np.eye(k)).max() <= 1e-12
    for (ell, r2), ho in zip(hist, o.hist):
        assert ell == ho[0] and abs(r2 - ho[2]) <= 1e-12 * nA ** 2


def test_shard_columns_partition():
    for n, P in [(10, 3), (20000, 8), (300, 2), (7, 7)]:
        parts = [shard_columns(n, P, r) for r in range(P)]
        assert parts[0][0] == 0
        for (o1, n1), (o2, _) in zip(parts, parts[1:]):
            assert o1 + n1 == o2
        assert sum(n for _, n in parts) == n
        assert max(n for _, n in parts) - min(n for _, n in parts) <= 1
    with pytest.raises(ValueError):
        shard_columns(3, 4, 0)


def test_nccl_unique_id_available_on_host():
    import paper_1503_07157_b200 as qbp
    try:
        uid = qbp.qb_nccl_unique_id()
    except qbp.QBError:
        pytest.skip("libnccl.so.2 not loadable here")
    assert len(uid) == 128 and any(uid)
