"""Time the FP32 downdate GEMM (C4 shape: A -= Q B, 200000 x 2000, K = 128) with CUDA events.

Usage: QB_LIB_PATH=<variant .so> python tools/tf32_down_time.py [w]
"""
import sys

import torch

import paper_1503_07157_b200 as qbp

m, n = 200000, 2000
w = int(sys.argv[1]) if len(sys.argv) > 1 else 128
c = qbp.QB(0, dtype=qbp.QB_F32)
A = torch.randn(n, m, device="cuda")
Q = torch.randn(w, m, device="cuda") / 400
Bt = torch.randn(w, n, device="cuda")
for _ in range(5):
    qbp.qb_gemm(c.ctx, 0, 2, m, n, w, Q.data_ptr(), m, Bt.data_ptr(), n, A.data_ptr(), m)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 20
e0.record()
for _ in range(R):
    qbp.qb_gemm(c.ctx, 0, 2, m, n, w, Q.data_ptr(), m, Bt.data_ptr(), n, A.data_ptr(), m)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
byts = 2 * m * n * 4 + m * w * 4 + w * n * 4
print(f"{qbp.LIB_PATH.split('/')[-1]} w={w} downdate {ms:.4f} ms  {byts / ms / 1e6:.0f} GB/s")
