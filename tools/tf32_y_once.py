"""Run the FP32 sketch GEMM Y = A Omega (C4 shape) a few times, for ncu captures."""
import torch

import paper_1503_07157_b200 as qbp

m, n, w = 200000, 2000, 128
c = qbp.QB(0, dtype=qbp.QB_F32)
A = torch.randn(n, m, device="cuda")            # col-major m x n
Om = torch.randn(n, w, device="cuda")           # row-major n x w
Y = torch.empty(w, m, dtype=torch.float64, device="cuda")
for _ in range(3):
    qbp.qb_gemm(c.ctx, 0, 0, m, w, n, A.data_ptr(), m, Om.data_ptr(), w, Y.data_ptr(), m)
torch.cuda.synchronize()
print("ok")
