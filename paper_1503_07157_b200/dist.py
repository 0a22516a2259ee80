"""Sharding of A across ranks.

Columns (square A): rank p of P owns the contiguous column block A(:, off_p : off_p + n_p).
The library draws the matching rows of every Ω_i from global indices, allreduces
Y_i = sum_p A_p Ω_p (and the Gram of the row-distributed power-step Z, and the norm scalars)
with NCCL, replicates the orth / re-projection, and keeps B_i and the downdate local.

Rows (tall-skinny A, NEXT-2): rank p owns A(off_p : off_p + m_p, :).  Ω is replicated, Y_i and
Q_i stay local; the CholeskyQR Grams, the re-projection W, the power step's Z and B_i are
allreduced, so B is replicated and Q is row-distributed.

torch.distributed is only the bootstrap: it carries the 128-byte ncclUniqueId from rank 0 to
the others.
"""


def shard_columns(n, nranks, rank):
    """(offset, count) of a balanced contiguous split of n columns (or rows) over nranks."""
    if nranks < 1 or not 0 <= rank < nranks or n < nranks:
        raise ValueError(f"cannot split {n} columns over {nranks} ranks (rank {rank})")
    base, extra = divmod(n, nranks)
    off = rank * base + min(rank, extra)
    return off, base + (1 if rank < extra else 0)


def broadcast_unique_id(uid, group=None):
    """Broadcast rank 0's 128-byte id with torch.distributed (any backend)."""
    import torch
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend(group) == "gloo" else f"cuda:{torch.cuda.current_device()}"
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == 0:
        t.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().tolist())


shard_rows = shard_columns


def dist_spec_rows(m_global, group=None):
    """dict(shard="rows", rank, nranks, unique_id, row_offset, m_local, m_global) for this process."""
    import torch.distributed as dist
    import paper_1503_07157_b200 as qbp
    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    uid = qbp.qb_nccl_unique_id() if rank == 0 else bytes(128)
    uid = broadcast_unique_id(uid, group)
    off, ml = shard_rows(m_global, nranks, rank)
    return dict(shard="rows", rank=rank, nranks=nranks, unique_id=uid, row_offset=off, m_local=ml,
                m_global=m_global)


def dist_spec(n_global, group=None):
    """dict(rank, nranks, unique_id, col_offset, n_local, n_global) for this process."""
    import torch.distributed as dist
    import paper_1503_07157_b200 as qbp
    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    uid = qbp.qb_nccl_unique_id() if rank == 0 else bytes(128)
    uid = broadcast_unique_id(uid, group)
    off, nl = shard_columns(n_global, nranks, rank)
    return dict(rank=rank, nranks=nranks, unique_id=uid, col_offset=off, n_local=nl, n_global=n_global)
