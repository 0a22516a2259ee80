"""Seeded synthetic inputs shared by tests, bench.py and smoke().

This module holds none of the method's arithmetic: it only builds test matrices
A = U diag(σ) V^* with orthonormal U, V "obtained by performing qr on a random Gaussian
matrix" (the paper's test-matrix recipe) and the spectra of the
BASELINE.json configs.  Both the oracle and the CUDA path consume what it returns; neither
side's code lives here.

Small matrices are built on the CPU with numpy (PCG64 seeded), large ones on the GPU with
torch (Philox seeded, cuSOLVER QR) — a generator, not the product path.
"""
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    dtype: str          # "f64" | "f32"
    spectrum: str       # see sigma()
    rank: int           # number of nonzero singular values r
    eps: float          # absolute Frobenius tolerance
    b: int
    q: int
    seed_matrix: int
    seed_omega: int = 1


def sigma(kind, r):
    """Singular values σ_1..σ_r (j = 1-based).

    exp10_20   σ_j = 10^(-j/20)     BASELINE configs[0]
    poly2      σ_j = j^-2           BASELINE configs[1] (paper-like polynomial decay)
    exp10_125  σ_j = 10^(-j/125)    configs[2] "fast decay" (reading)
    exp_100    σ_j = e^(-j/100)     configs[3]
    exp_150    σ_j = e^(-j/150)     configs[4] and the 20000^2 target "slow decay"
    matrix1    σ_j = g_j^2 0.65^(j-1), g_j ~ U[0,1]  (Matrix 1; needs rng)
    """
    j = np.arange(1, r + 1, dtype=np.float64)
    if kind == "exp10_20":
        return 10.0 ** (-j / 20.0)
    if kind == "poly2":
        return j ** -2.0
    if kind == "exp10_125":
        return 10.0 ** (-j / 125.0)
    if kind == "exp_100":
        return np.exp(-j / 100.0)
    if kind == "exp_150":
        return np.exp(-j / 150.0)
    raise ValueError(kind)


CONFIGS = {
    # BASELINE.json configs, in order; "T" is the north_star target (20000^2, b = 256).
    "C1": Config("C1", 400, 300, "f64", "exp10_20", 300, 1e-6, 10, 0, 1000),
    "C2": Config("C2", 4000, 4000, "f64", "poly2", 4000, 1e-4, 64, 0, 1001),
    "C3": Config("C3", 10000, 10000, "f64", "exp10_125", 10000, 1e-8, 128, 1, 1002),
    "C4": Config("C4", 200000, 2000, "f32", "exp_100", 2000, 1e-3, 128, 0, 1003),
    "C5": Config("C5", 50000, 50000, "f64", "exp_150", 3584, 1e-6, 256, 1, 1004),
    "T": Config("T", 20000, 20000, "f64", "exp_150", 20000, 1e-6, 256, 0, 1005),
    "T1": Config("T1", 20000, 20000, "f64", "exp_150", 20000, 1e-6, 256, 1, 1005),
}


def eps_rank(sig, eps):
    """k_ε = min{k : sum_{j>k} σ_j^2 <= ε^2} (Eckart-Young)."""
    sig = np.sort(np.asarray(sig, dtype=np.float64))[::-1]
    tail = np.concatenate([np.cumsum((sig ** 2)[::-1])[::-1], [0.0]])  # tail[k] = sum_{j>k}
    return int(np.argmax(tail <= eps * eps))


def optimal_error(sig, k):
    """min over rank-k B of ||A - B||_F = (sum_{j>k} σ_j^2)^(1/2)."""
    sig = np.sort(np.asarray(sig, dtype=np.float64))[::-1]
    return float(np.sqrt(np.sum(sig[k:] ** 2)))


def haar_np(rng, m, r):
    """m x r matrix with orthonormal columns: economy QR of a Gaussian matrix."""
    Q, R = np.linalg.qr(rng.standard_normal((m, r)))
    return Q * np.sign(np.diag(R))[None, :]


def make_matrix_np(m, n, sig, seed):
    """A = U diag(σ) V^* (float64, Fortran order) built on the CPU."""
    rng = np.random.default_rng(seed)
    r = len(sig)
    U = haar_np(rng, m, r)
    V = haar_np(rng, n, r)
    return np.asfortranarray((U * sig[None, :]) @ V.T)


def make_matrix_torch(m, n, sig, seed, device="cuda", dtype=None):
    """A = U diag(σ) V^* built on `device` with torch; returned column-major
    (a transposed view of a contiguous n x m tensor, so A[i, j] sits at i + j*m)."""
    import torch
    dtype = dtype or torch.float64
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    r = len(sig)
    s = torch.as_tensor(np.asarray(sig), dtype=torch.float64, device=device)
    U, _ = torch.linalg.qr(torch.randn(m, r, generator=g, dtype=torch.float64, device=device))
    V, _ = torch.linalg.qr(torch.randn(n, r, generator=g, dtype=torch.float64, device=device))
    At = (V * s[None, :]) @ U.T          # n x m contiguous = A^T
    del U, V
    return At.to(dtype).t()


def make_shard_torch(m, n_local, sig, seed, rank, nranks, device="cuda", dtype=None):
    """Column block `rank` of the m x (nranks * n_local) matrix
    A = U diag(σ) [V_0; ...; V_{P-1}]^T / sqrt(P), each V_p an n_local x r orthonormal factor.
    The stacked right factor has orthonormal columns (sum_p V_p^T V_p / P = I), so A has
    exactly the singular values σ for every P, and rank 0 of P = 1 is make_matrix_torch.
    Used for weak scaling: every rank holds an m x n_local block."""
    import torch
    dtype = dtype or torch.float64
    r = len(sig)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    s = torch.as_tensor(np.asarray(sig), dtype=torch.float64, device=device) / np.sqrt(nranks)
    U, _ = torch.linalg.qr(torch.randn(m, r, generator=g, dtype=torch.float64, device=device))
    if rank > 0:
        g = torch.Generator(device=device)
        g.manual_seed(int(seed) * 1000003 + int(rank))
    V, _ = torch.linalg.qr(torch.randn(n_local, r, generator=g, dtype=torch.float64, device=device))
    At = (V * s[None, :]) @ U.T
    del U, V
    return At.to(dtype).t()


def make_row_shard_torch(m_local, n, sig, seed, rank, nranks, device="cuda", dtype=None):
    """Row block `rank` of the (nranks * m_local) x n matrix
    A = [U_0; ...; U_{P-1}] diag(σ) V^T / sqrt(P), each U_p an m_local x r orthonormal factor:
    the stacked left factor has orthonormal columns, so A has exactly the singular values σ for
    every P (the row-sharded analogue of make_shard_torch, for tall-skinny weak scaling)."""
    import torch
    dtype = dtype or torch.float64
    r = len(sig)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    s = torch.as_tensor(np.asarray(sig), dtype=torch.float64, device=device) / np.sqrt(nranks)
    V, _ = torch.linalg.qr(torch.randn(n, r, generator=g, dtype=torch.float64, device=device))
    if rank > 0:
        g = torch.Generator(device=device)
        g.manual_seed(int(seed) * 1000003 + int(rank))
    U, _ = torch.linalg.qr(torch.randn(m_local, r, generator=g, dtype=torch.float64, device=device))
    At = (V * s[None, :]) @ U.T          # n x m_local contiguous = A_p^T
    del U, V
    return At.to(dtype).t()


def config_sigma(cfg):
    return sigma(cfg.spectrum, cfg.rank)


def random_matrix_np(m, n, seed):
    """Plain Gaussian test matrix (kernel-level parity tests)."""
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((m, n)))
