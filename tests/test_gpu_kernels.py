"""Kernel-level GPU tests through the C ABI test hooks: the FP64 GEMM (every contraction of the
loop) against a plain FP64 product on ragged shapes, every layout and epilogue, split and
unsplit; bitwise run-to-run reproducibility of the GEMM and of CholeskyQR (fixed-order
reductions)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def q():
    import paper_1503_07157_b200 as qbp
    from paper_1503_07157_b200 import build
    build.build()
    c = qbp.QB(0)
    yield qbp, c
    c.close()


def dev_colmajor(X, ld=None):
    """Column-major device copy with leading dimension ld (>= rows, even)."""
    r, c = X.shape
    ld = ld or (r + (r & 1))
    buf = torch.zeros((c, ld), dtype=torch.float64, device="cuda")
    buf[:, :r] = torch.from_numpy(np.ascontiguousarray(X.T))
    return buf, ld


def from_colmajor(buf, r):
    return buf[:, :r].T.cpu().numpy()


SHAPES = [(1, 1, 1), (7, 5, 3), (128, 64, 16), (129, 65, 17), (300, 200, 1000), (1000, 256, 5000),
          (256, 20000 // 16, 333), (4000, 130, 64), (200, 2100, 40), (385, 4096, 256)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_matches_fp64_product(q, M, N, K, layout, epi):
    qbp, c = q
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    Am = rng.standard_normal((M, K))     # op(A): M x K
    Bm = rng.standard_normal((K, N))     # op(B): K x N
    if layout == 0:   # A M-contiguous (column-major M x K), B N-contiguous (row-major K x N)
        A, lda = dev_colmajor(Am)
        B, ldb = dev_colmajor(Bm.T)
    else:             # A K-contiguous (column-major K x M), B K-contiguous (column-major K x N)
        A, lda = dev_colmajor(Am.T)
        B, ldb = dev_colmajor(Bm)
    ref = Am @ Bm
    C0 = rng.standard_normal((M, N))
    if epi == 1:
        C, ldc = dev_colmajor(C0.T)      # row-major M x N == column-major N x M
    else:
        C, ldc = dev_colmajor(C0)
    for split in (False, True):
        Cw = C.clone()
        ss = qbp.qb_gemm(c.ctx, layout, epi, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, Cw.data_ptr(), ldc,
                         split=split, want_sumsq=True)
        got = from_colmajor(Cw, N).T if epi == 1 else from_colmajor(Cw, M)
        want = C0 - ref if epi == 2 else ref
        scale = np.sqrt(K) * 1e-15 * (np.abs(Am) @ np.abs(Bm)).max() + 1e-300
        assert np.abs(got - want).max() <= 8 * scale, (split, np.abs(got - want).max(), scale)
        assert abs(ss - float(np.sum(want * want))) <= 1e-12 * float(np.sum(want * want)) + 1e-300
        # padding rows between M (or N) and ld untouched
        if epi != 1 and ldc > M:
            assert torch.equal(Cw[:, M:], C[:, M:])


def test_gemm_bitwise_reproducible(q):
    qbp, c = q
    rng = np.random.default_rng(1)
    M, N, K = 20000, 256, 20000
    A = torch.from_numpy(rng.standard_normal((K, M))).cuda()      # column-major M x K: A[i + k*M]
    B = torch.from_numpy(rng.standard_normal((K, N))).cuda()      # row-major K x N
    outs = []
    for _ in range(4):
        C = torch.empty((N, M), dtype=torch.float64, device="cuda")
        qbp.qb_gemm(c.ctx, 0, 0, M, N, K, A.data_ptr(), M, B.data_ptr(), N, C.data_ptr(), M)
        outs.append(C)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_orth_bitwise_reproducible(q):
    qbp, c = q
    X = torch.from_numpy(np.random.default_rng(2).standard_normal((256, 20000))).cuda()  # col-major 20000 x 256
    outs = []
    for _ in range(6):
        Y = X.clone()
        qbp.qb_orth(c.ctx, Y.data_ptr(), 20000, 256, 20000)
        outs.append(Y)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("w", [1, 5, 32, 33, 64, 100, 255, 256])
def test_chol_rinv_parity_and_reproducible(q, w):
    qbp, c = q
    rng = np.random.default_rng(w)
    X = rng.standard_normal((4 * w + 7, w)) * np.exp(-np.arange(w) / 60.0)[None, :]
    G = X.T @ X
    Gd = torch.from_numpy(G.T.copy()).cuda()           # column-major
    outs = []
    for _ in range(5):
        R = torch.zeros((w, w), dtype=torch.float64, device="cuda")
        sh = qbp.qb_chol_rinv(c.ctx, Gd.data_ptr(), w, w, X.shape[0], R.data_ptr(), w)
        assert sh == 0
        outs.append(R)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    Rinv = outs[0].cpu().numpy()                       # row-major w x w
    Rref = np.linalg.inv(np.linalg.cholesky(G).T)
    assert np.allclose(np.triu(Rinv), Rinv)
    assert np.abs(Rinv - Rref).max() <= 1e-10 * np.abs(Rref).max()
    Q = X @ Rinv
    assert np.abs(Q.T @ Q - np.eye(w)).max() <= 1e-9


def test_gram_gemm_bitwise_reproducible(q):
    qbp, c = q
    X = torch.from_numpy(np.random.default_rng(3).standard_normal((256, 20000))).cuda()  # col-major 20000 x 256
    outs = []
    for _ in range(5):
        G = torch.empty((256, 256), dtype=torch.float64, device="cuda")
        qbp.qb_gemm(c.ctx, 1, 0, 256, 256, 20000, X.data_ptr(), 20000, X.data_ptr(), 20000, G.data_ptr(), 256)
        outs.append(G)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("M,N,K", [(2000, 20000, 256), (1990, 19970, 130), (300, 40000, 64)])
def test_persistent_downdate_matches_fp64(q, M, N, K):
    """The persistent subtract-update (TMEM-parked accumulators, epilogue hidden under the next
    tile) that runs the downdate A -= Q_i B_i: ragged M and N, nk >= 16 and 8 <= nk < 16."""
    qbp, c = q
    rng = np.random.default_rng(M + N + K)
    Qm = rng.standard_normal((M, K)) / np.sqrt(K)
    Bm = rng.standard_normal((K, N))
    C0 = rng.standard_normal((M, N))
    A, lda = dev_colmajor(Qm)
    B, ldb = dev_colmajor(Bm.T)
    C, ldc = dev_colmajor(C0)
    outs = []
    for _ in range(2):
        Cw = C.clone()
        ss = qbp.qb_gemm(c.ctx, 0, 2, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, Cw.data_ptr(), ldc,
                         split=False, want_sumsq=True)
        outs.append((Cw, ss))
    assert torch.equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]
    got = from_colmajor(outs[0][0], M)
    want = C0 - Qm @ Bm
    scale = np.sqrt(K) * 1e-15 * (np.abs(Qm) @ np.abs(Bm)).max()
    assert np.abs(got - want).max() <= 8 * scale + 1e-15
    assert abs(outs[0][1] - float(np.sum(want * want))) <= 1e-12 * float(np.sum(want * want))
