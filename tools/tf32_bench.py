"""Time the FP32 (3xTF32 tcgen05) GEMM on the C4 loop shapes through qb_gemm (CUDA events).

    PYTHONPATH=. python tools/tf32_bench.py
"""
import sys

import torch

import paper_1503_07157_b200 as qbp


def bench(c, layout, epi, M, N, K, A, lda, B, ldb, C, ldc, reps=10):
    qbp.qb_gemm(c.ctx, layout, epi, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), ldc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        qbp.qb_gemm(c.ctx, layout, epi, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), ldc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 2.0 * M * N * K
    return ms, fl / ms / 1e9


def main():
    m, n, w = 200000, 2000, 128
    c = qbp.QB(0, dtype=qbp.QB_F32)
    A = torch.randn(n, m, device="cuda")            # col-major m x n
    Om = torch.randn(n, w, device="cuda")           # row-major n x w
    Q = torch.randn(w, m, device="cuda") / 400      # col-major m x w
    Bt = torch.randn(w, n, device="cuda")           # row-major w x n
    Y = torch.empty(w, m, dtype=torch.float64, device="cuda")
    Bo = torch.empty(w, n, dtype=torch.float64, device="cuda")
    rows = []
    ms, tf = bench(c, 0, 0, m, w, n, A, m, Om, w, Y, m)
    rows.append(("Y = A Om   (NN, store)", ms, tf))
    ms, tf = bench(c, 1, 1, w, n, m, Q, m, A, m, Bo, n)
    rows.append(("B = Q^T A  (TN, row, split)", ms, tf))
    ms, tf = bench(c, 0, 2, m, n, w, Q, m, Bt, n, A, m)
    rows.append(("A -= Q B   (NN, sub)", ms, tf))
    for name, ms, tf in rows:
        print(f"{name:32s} {ms:8.3f} ms  {tf:8.1f} TFLOP/s (FP32-equivalent)")
    sys.stdout.flush()


if __name__ == "__main__":
    main()
