"""Run the FP32 downdate GEMM (C4 shape) a few times, for ncu captures."""
import torch

import paper_1503_07157_b200 as qbp

m, n, w = 200000, 2000, 128
c = qbp.QB(0, dtype=qbp.QB_F32)
A = torch.randn(n, m, device="cuda")
Q = torch.randn(w, m, device="cuda") / 400
Bt = torch.randn(w, n, device="cuda")
for _ in range(3):
    qbp.qb_gemm(c.ctx, 0, 2, m, n, w, Q.data_ptr(), m, Bt.data_ptr(), n, A.data_ptr(), m)
torch.cuda.synchronize()
print("ok")
