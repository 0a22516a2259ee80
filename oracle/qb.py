"""Oracle: the blocked adaptive randomized QB factorization, step by step (TEST INFRASTRUCTURE;
see oracle/__init__.py).  FP64 numpy; every matrix product is one ``@`` (a library GEMM, a
permitted primitive) and ``orth`` is a packaged economy QR, exactly as the paper defines it.

Paper references are PAPER.md line numbers:
  problem statement           :19-25, :39-46, Algorithm 1 :91-121
  Frobenius norm (default)    :186-188
  orth(X) = qr(X, 0)          :281-292
  randQB (Fig. 1, unblocked)  :319-337
  blocking (def0)-(def3)      :474-505
  randQB_b (Fig. 2)           :698-725
  randQB_p (Fig. 3)           :826-849
  randQB_pb (Fig. 4)          :859-887
  QB -> partial SVD           :390-406
Readings where the paper is silent or garbled (R1-R20) are listed in DESIGN.md §3.
"""
from dataclasses import dataclass, field

import numpy as np

from .omega import omega_panel

QB_OK = 0
QB_NOT_CONVERGED = 1


def frob2(X):
    """||X||_F^2 = sum_ij |X(i,j)|^2, accumulated in FP64."""
    X = np.asarray(X, dtype=np.float64)
    return float(np.sum(X * X))


def orth(X):
    """orth(X): an orthonormal basis of ran(X) with as many columns as X, computed by an
    economy QR without pivoting ("Q = qr(X,0)").  The paper fixes no sign;
    reading R7 normalises the basis so that diag(R) >= 0 (the CUDA CholeskyQR2 has
    diag(R) > 0 by construction), which makes the basis unique for full-rank X."""
    Q, R = np.linalg.qr(np.asarray(X, dtype=np.float64), mode="reduced")
    d = np.sign(np.diag(R))
    d[d == 0] = 1.0
    return Q * d[None, :]


def omega(seed, n, col0, w, dtype=np.float64):
    """Ω_i = randn(n, w) for global columns col0 .. col0+w-1;
    reading R14/R15: the counter-based generator of DESIGN.md §3.3.  For the FP32 path the
    matrix is RN_32 of the FP64 draw (reading R18), returned widened back to FP64."""
    O = omega_panel(seed, n, col0, w)
    if dtype == np.float32:
        O = O.astype(np.float32).astype(np.float64)
    return O


@dataclass
class QBResult:
    status: int
    k: int
    Q: np.ndarray           # m x k, orthonormal columns
    B: np.ndarray           # k x n
    r2_0: float             # ||A||_F^2
    hist: list = field(default_factory=list)   # per block: (ell, w, r2 = ||A^(i)||_F^2, EI)

    @property
    def resid(self):
        return float(np.sqrt(self.hist[-1][2])) if self.hist else float(np.sqrt(self.r2_0))


def randqb_pb(A, eps, b, q=0, seed=1, kmax=None, reproj=True, omega_dtype=np.float64, skip_power_orth=False):
    """randQB_pb (Fig. 4) with P = q power steps; q = 0 is exactly
    randQB_b (Fig. 2).

    A (m x n) is copied: A^(0) = A (eq. (def0), :494), and A^(i) overwrites A^(i-1) (:112).
    eps is the absolute Frobenius tolerance (reading R2).  The loop stops after the first
    block whose residual satisfies ||A^(i)||_F^2 <= eps^2 (Fig. 2 line (6), reading R4 for
    "<" vs "<="), checked on the directly computed residual (reading R1); the error
    indicator EI_i = ||A||_F^2 - sum_j ||B_j||_F^2 is recorded beside it.  Before the first
    block, ||A||_F <= eps returns k = 0 (Algorithm 1 line (2), reading R3).  kmax caps the
    rank; the last block is narrowed to hit it (reading R5).

    skip_power_orth: the variant of PAPER.md:915-931 ("Is re-orthonormalizing truly
    necessary?") applied per block: Y = A Ω; q times Y = A (A^* Y); Q_i = orth(Y).
    """
    A = np.array(A, dtype=np.float64, copy=True)          # A^(0) = A
    m, n = A.shape
    kmax = min(m, n) if kmax is None or kmax <= 0 else min(int(kmax), m, n)
    eps2 = float(eps) * float(eps)
    r2 = frob2(A)
    res = QBResult(QB_OK, 0, np.zeros((m, 0)), np.zeros((0, n)), r2)
    if r2 <= eps2:
        return res
    Qs, Bs = [], []
    ei = r2
    ell = 0
    while ell < kmax:
        w = min(b, kmax - ell)
        Om = omega(seed, n, ell, w, omega_dtype)                     # line (2)
        if skip_power_orth:
            Y = A @ Om
            for _ in range(q):
                Y = A @ (A.T @ Y)
            Qi = orth(Y)
        else:
            Qi = orth(A @ Om)                                        # line (3)
            for _ in range(q):                                       # lines (4)-(7)
                Qi = orth(A.T @ Qi)                                  # line (5)
                Qi = orth(A @ Qi)                                    # line (6)
        if ell > 0 and reproj:                                       # line (8) / (3')
            Qbar = np.hstack(Qs)
            Qi = orth(Qi - Qbar @ (Qbar.T @ Qi))
        Bi = Qi.T @ A                                                # line (9) / (4)
        A = A - Qi @ Bi                                              # line (10) / (5)
        r2 = frob2(A)                                                # ||A^(i)||_F^2
        ei = ei - frob2(Bi)                                          # error indicator
        Qs.append(Qi)
        Bs.append(Bi)
        ell += w
        res.hist.append((ell, w, r2, ei))
        if r2 <= eps2:                                               # line (11) / (6)
            break
    res.status = QB_OK if r2 <= eps2 else QB_NOT_CONVERGED
    res.k = ell
    res.Q = np.hstack(Qs)
    res.B = np.vstack(Bs)
    return res


def randqb(A, ell, seed=1, omega_dtype=np.float64):
    """randQB (Fig. 1), the unblocked fixed-rank scheme:
    Ω = randn(n, ℓ); Q = orth(AΩ); B = Q^* A.  Ω is columns 0..ℓ-1 of the same generator,
    so its slices are the Ω_i of the blocked scheme (eq. (OmegaBlock), :479-484).
    omega_dtype=np.float32: Ω = RN_32(Ω) (reading R18), arithmetic still FP64."""
    A = np.asarray(A, dtype=np.float64)
    Q = orth(A @ omega(seed, A.shape[1], 0, ell, omega_dtype))
    return Q, Q.T @ A


def randqb_p(A, ell, P, seed=1, skip_power_orth=False, omega_dtype=np.float64):
    """randQB_p (Fig. 3): Q = orth(AΩ); P times {Q = orth(A^*Q);
    Q = orth(AQ)}; B = Q^* A.  skip_power_orth: Y = AΩ; P times Y = A(A^*Y); Q = orth(Y)
    (PAPER.md:919-927).  omega_dtype as in randqb."""
    A = np.asarray(A, dtype=np.float64)
    if skip_power_orth:
        Y = A @ omega(seed, A.shape[1], 0, ell, omega_dtype)
        for _ in range(P):
            Y = A @ (A.T @ Y)
        Q = orth(Y)
        return Q, Q.T @ A
    Q = orth(A @ omega(seed, A.shape[1], 0, ell, omega_dtype))
    for _ in range(P):
        Q = orth(A.T @ Q)
        Q = orth(A @ Q)
    return Q, Q.T @ A


def qb_to_svd(Q, B):
    """QB -> partial SVD: B = Û D V^*, U = Q Û; A ≈ U D V^*."""
    Uh, D, Vt = np.linalg.svd(np.asarray(B, dtype=np.float64), full_matrices=False)
    return Q @ Uh, D, Vt.T


def tail_rank(D, resid2, eps=0.0, kkeep=0):
    """The rank kept when converting a QB factorization with residual ||A - QB||_F^2 = resid2 to a
    partial SVD with singular values D (descending): "choose a rank k ... based on the decaying
    singular values"; truncating the SVD of B to k' terms adds exactly the
    dropped D_j^2 to the squared error, ||A - U_k' D_k' V_k'^*||_F^2 = resid2 + sum_{j >= k'} D_j^2
    (the SVD tail identity), so k' = the smallest rank with that error <= eps^2 (eps > 0), capped
    by kkeep (> 0).  The sum runs from the smallest D_j up, as written."""
    D = np.asarray(D, dtype=np.float64)
    k = len(D)
    kk = k
    if eps > 0:
        tail = float(resid2)
        for j in range(k - 1, -1, -1):
            nt = tail + D[j] * D[j]
            if nt > eps * eps:
                break
            tail = nt
            kk = j
    if kkeep > 0:
        kk = min(kk, int(kkeep))
    return kk


def qb_to_svd_truncated(Q, B, resid2, eps=0.0, kkeep=0):
    """QB -> partial SVD truncated to tail_rank(D, resid2, eps, kkeep) triplets."""
    U, D, V = qb_to_svd(Q, B)
    kk = tail_rank(D, resid2, eps, kkeep)
    return U[:, :kk], D[:kk], V[:, :kk]


def pivoted_qr(B):
    """QB -> partial pivoted QR: B P = Q~ R by Householder QR with column
    pivoting, step by step in LAPACK dlaqp2's order (the order the paper's "pivoted QR" refers to,
    P:242-279): at step i the pivot is the FIRST column of largest partial norm; the reflector
    H_i = I - tau v v^T has v_0 = 1 and beta = -sign(alpha) ||x|| (dlarfg; tau = 0 when x below the
    diagonal is zero); it is applied to the trailing columns; the partial norms are downdated with
    R(i, j) and recomputed from scratch when the sqrt(eps) cancellation test fires.
    Returns (perm, Q~ (l x l), R (l x n upper trapezoidal)): column j of B P is column perm[j] of B."""
    R = np.array(B, dtype=np.float64, copy=True)
    l, n = R.shape
    kmin = min(l, n)
    perm = np.arange(n)
    vn1 = np.sqrt(np.sum(R * R, axis=0))
    vn2 = vn1.copy()
    tol3z = np.sqrt(np.finfo(np.float64).eps)
    taus, vs = [], []
    for i in range(kmin):
        p = i + int(np.argmax(vn1[i:]))
        if p != i:
            R[:, [i, p]] = R[:, [p, i]]
            perm[[i, p]] = perm[[p, i]]
            vn1[p], vn2[p] = vn1[i], vn2[i]
        alpha = R[i, i]
        x = R[i + 1:, i].copy()
        xnorm = float(np.sqrt(np.sum(x * x)))
        v = np.zeros(l - i)
        v[0] = 1.0
        if xnorm == 0.0:
            tau, beta = 0.0, alpha
        else:
            beta = -np.copysign(np.hypot(alpha, xnorm), alpha)
            tau = (beta - alpha) / beta
            v[1:] = x / (alpha - beta)
        R[i, i] = beta
        R[i + 1:, i] = 0.0
        if tau != 0.0 and i + 1 < n:
            w = v @ R[i:, i + 1:]
            R[i:, i + 1:] -= tau * np.outer(v, w)
        for j in range(i + 1, n):
            if vn1[j] != 0.0:
                temp = max(0.0, 1.0 - (abs(R[i, j]) / vn1[j]) ** 2)
                temp2 = temp * (vn1[j] / vn2[j]) ** 2
                if temp2 <= tol3z:
                    vn1[j] = float(np.sqrt(np.sum(R[i + 1:, j] ** 2))) if i + 1 < l else 0.0
                    vn2[j] = vn1[j]
                else:
                    vn1[j] *= np.sqrt(temp)
        taus.append(tau)
        vs.append(v)
    Q = np.eye(l)
    for i in range(kmin - 1, -1, -1):          # Q~ = H_0 H_1 ... H_{k-1}, applied to the identity
        v = vs[i]
        Q[i:, :] -= taus[i] * np.outer(v, v @ Q[i:, :])
    return perm, Q, np.triu(R)
