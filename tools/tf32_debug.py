"""Diagnose the tcgen05 TF32 GEMM on small integer problems (prints error summaries).

    PYTHONPATH=. python tools/tf32_debug.py
"""
import numpy as np
import torch

import paper_1503_07157_b200 as qbp

np.set_printoptions(linewidth=200, precision=1, suppress=True)


def dev(X, dtype):
    r, c = X.shape
    ld = (r + 3) // 4 * 4
    buf = torch.zeros((c, ld), dtype=dtype, device="cuda")
    buf[:, :r] = torch.from_numpy(np.ascontiguousarray(X.T)).to(dtype)
    return buf, ld


def main():
    c = qbp.QB(0, dtype=qbp.QB_F32)
    for (M, N, K) in [(128, 64, 32), (128, 64, 8), (1, 1, 1), (128, 128, 64), (256, 256, 256)]:
        for layout in (0, 1):
            rng = np.random.default_rng(0)
            if K == 8 or M == 1:
                Am = np.zeros((M, K)); Bm = np.zeros((K, N))
                Am[:, 0] = np.arange(M) % 7 + 1
                Bm[0, :] = np.arange(N) % 5 + 1
            else:
                Am = rng.integers(-3, 4, (M, K)).astype(np.float64)
                Bm = rng.integers(-3, 4, (K, N)).astype(np.float64)
            if layout == 0:
                A, lda = dev(Am, torch.float32)
                B, ldb = dev(Bm.T, torch.float32)
            else:
                A, lda = dev(Am.T, torch.float32)
                B, ldb = dev(Bm, torch.float32)
            C, ldc = dev(np.zeros((M, N)), torch.float64)
            qbp.qb_gemm(c.ctx, layout, 0, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), ldc,
                        split=False)
            got = C[:, :M].T.cpu().numpy()
            want = Am @ Bm
            err = np.abs(got - want)
            print(f"M={M} N={N} K={K} layout={layout}: maxerr {err.max():.3g}  nnz(got) {np.count_nonzero(got)}"
                  f" nnz(want) {np.count_nonzero(want)} sum got {got.sum():.6g} want {want.sum():.6g}")
            if err.max() > 0 and M >= 8 and N >= 8:
                print(" got[:8,:8]\n", got[:8, :8], "\n want[:8,:8]\n", want[:8, :8])
                bad = np.argwhere(err > 0)
                print(" first bad", bad[:10].tolist(), "count", len(bad))
                # is got a permutation of rows/cols of want?
                if K == 8:
                    print(" got row sums", got.sum(1)[:16], "\n want row sums", want.sum(1)[:16])


if __name__ == "__main__":
    main()
