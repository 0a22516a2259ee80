"""Kernel-level GPU tests of the FP32 GEMM (tcgen05.mma kind::tf32, 3xTF32 split, TMEM
accumulators; csrc/gemm_tf32.cuh) through the qb_gemm test hook on an FP32 context.

  * exactness: small-integer operands are exact in TF32 (lo = 0) and their K-term sums are
    exact in FP32, so any layout / descriptor / swizzle / epilogue mistake shows as a nonzero
    difference — the result must equal the FP64 product bit for bit;
  * accuracy: Gaussian operands against the FP64 product, with the FP32 bound of DESIGN.md
    reading R18b (|err_ij| <= (K 2^-24 + 3 2^-21)(|A||B|)_ij) and a Frobenius relative error far
    below what a single TF32 product would give (which would be ~1e-4);
  * every layout x epilogue, ragged M / N / K, split and unsplit, bitwise reproducibility."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def q():
    import paper_1503_07157_b200 as qbp
    from paper_1503_07157_b200 import build
    build.build()
    c = qbp.QB(0, dtype=qbp.QB_F32)
    yield qbp, c
    c.close()


def dev_colmajor(X, dtype, ld=None):
    """Column-major device copy (leading dimension a multiple of 4: 16-byte TMA rows)."""
    r, c = X.shape
    ld = ld or ((r + 3) // 4 * 4)
    buf = torch.zeros((c, ld), dtype=dtype, device="cuda")
    buf[:, :r] = torch.from_numpy(np.ascontiguousarray(X.T)).to(dtype)
    return buf, ld


def from_colmajor(buf, r):
    return buf[:, :r].T.double().cpu().numpy()


def operands(Am, Bm, layout):
    if layout == 0:   # A M-contiguous (col-major M x K), B N-contiguous (row-major K x N)
        A, lda = dev_colmajor(Am, torch.float32)
        B, ldb = dev_colmajor(Bm.T, torch.float32)
    else:             # A K-contiguous (col-major K x M), B K-contiguous (col-major K x N)
        A, lda = dev_colmajor(Am.T, torch.float32)
        B, ldb = dev_colmajor(Bm, torch.float32)
    return A, lda, B, ldb


def run(qbp, c, layout, epi, M, N, K, A, lda, B, ldb, C0, split):
    if epi == 2:
        C, ldc = dev_colmajor(C0, torch.float32)
    elif epi == 1:
        C, ldc = dev_colmajor(C0.T, torch.float64)
    else:
        C, ldc = dev_colmajor(C0, torch.float64)
    ss = qbp.qb_gemm(c.ctx, layout, epi, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), ldc,
                     split=split, want_sumsq=True)
    got = from_colmajor(C, N).T if epi == 1 else from_colmajor(C, M)
    return got, ss, C, ldc


SHAPES = [(1, 1, 1), (7, 5, 3), (128, 64, 32), (129, 65, 33), (300, 200, 1000), (1000, 256, 5000),
          (256, 1250, 333), (4000, 130, 64), (200, 2100, 40), (385, 2000, 256), (2000, 128, 20000),
          # short K with >= 4 row tiles: the subtract-update keeps A's row block in TMEM
          # (several tiles per CTA share a row block in the last two)
          (1000, 300, 128), (777, 129, 100), (2000, 2000, 33), (513, 64, 1), (40000, 256, 128), (20000, 700, 96)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_tf32_gemm_exact_on_integers(q, M, N, K, layout, epi):
    qbp, c = q
    rng = np.random.default_rng(M * 7 + N * 3 + K + 11 * layout + epi)
    Am = rng.integers(-8, 9, (M, K)).astype(np.float64)
    Bm = rng.integers(-8, 9, (K, N)).astype(np.float64)
    if K > 2000:
        Am = np.clip(Am, -2, 2)
        Bm = np.clip(Bm, -2, 2)
    C0 = rng.integers(-100, 101, (M, N)).astype(np.float64)
    A, lda, B, ldb = operands(Am, Bm, layout)
    want = C0 - Am @ Bm if epi == 2 else Am @ Bm
    for split in (False, True):
        got, ss, _, _ = run(qbp, c, layout, epi, M, N, K, A, lda, B, ldb, C0, split)
        assert np.array_equal(got, want), (split, np.abs(got - want).max())
        # SUB_COL's fused sum of squares: FP32 over 8 entries, then FP64 (R18)
        ssw = float(np.sum(want * want))
        assert ss == ssw if epi != 2 else abs(ss - ssw) <= 8 * 2.0 ** -24 * ssw


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_tf32_gemm_fp32_accuracy(q, M, N, K, layout, epi):
    qbp, c = q
    rng = np.random.default_rng(M * 5 + N * 11 + K + 7 * layout + epi)
    Am = rng.standard_normal((M, K)).astype(np.float32).astype(np.float64)
    Bm = rng.standard_normal((K, N)).astype(np.float32).astype(np.float64)
    C0 = rng.standard_normal((M, N)).astype(np.float32).astype(np.float64)
    A, lda, B, ldb = operands(Am, Bm, layout)
    ref = Am @ Bm
    want = C0 - ref if epi == 2 else ref
    absprod = np.abs(Am) @ np.abs(Bm)
    bound = (K * 2.0 ** -24 + 3 * 2.0 ** -21) * absprod + (2.0 ** -24 * np.abs(want) if epi == 2 else 0)
    for split in (False, True):
        got, ss, C, ldc = run(qbp, c, layout, epi, M, N, K, A, lda, B, ldb, C0, split)
        err = np.abs(got - want)
        assert (err <= bound + 1e-30).all(), (split, (err / (bound + 1e-30)).max())
        rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
        assert rel <= 2e-6 * max(1.0, np.log2(K)), (split, rel)
        ssw = float(np.sum(got * got))
        assert abs(ss - ssw) <= (8 * 2.0 ** -24 if epi == 2 else 1e-12) * ssw + 1e-300
        if epi != 1 and ldc > M:      # padding rows between M and ld untouched
            assert not C[:, M:].any()


def test_tf32_gemm_bitwise_reproducible(q):
    qbp, c = q
    rng = np.random.default_rng(1)
    M, N, K = 20000, 128, 20000
    A = torch.from_numpy(rng.standard_normal((K, M)).astype(np.float32)).cuda()   # col-major M x K
    B = torch.from_numpy(rng.standard_normal((K, N)).astype(np.float32)).cuda()   # row-major K x N
    outs = []
    for _ in range(4):
        C = torch.empty((N, M), dtype=torch.float64, device="cuda")
        qbp.qb_gemm(c.ctx, 0, 0, M, N, K, A.data_ptr(), M, B.data_ptr(), N, C.data_ptr(), M)
        outs.append(C)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
