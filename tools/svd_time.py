"""Time rqb_svd on a config (development helper).  PYTHONPATH=. python tools/svd_time.py T"""
import sys
import time

import torch

import synth
import paper_1503_07157_b200 as qbp

name = sys.argv[1] if len(sys.argv) > 1 else "T"
cfg = synth.CONFIGS[name]
dt = torch.float32 if cfg.dtype == "f32" else torch.float64
A = synth.make_matrix_torch(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix, dtype=dt)
c = qbp.QB(0, dtype=qbp.QB_F32 if cfg.dtype == "f32" else qbp.QB_F64)
g = c.factor(A, cfg.eps, cfg.b, cfg.q, cfg.seed_omega, copy_out=False)
for r in range(2):
    torch.cuda.synchronize()
    t = time.time()
    s = c.svd(copy_out=False)
    torch.cuda.synchronize()
    dt_ms = (time.time() - t) * 1e3
    S = s["S"].double()
    ref = torch.exp(-torch.arange(1, g["k"] + 1, dtype=torch.float64, device="cuda") / 150.0)
    U = s["U"].double()
    print(f"{name} k={g['k']} svd {dt_ms:.1f} ms  max|S-sigma|[:k/2] {(S - ref)[:g['k'] // 2].abs().max().item():.3e}"
          f"  |U^TU-I| {(U.T @ U - torch.eye(g['k'], device='cuda', dtype=torch.float64)).abs().max().item():.2e}",
          flush=True)
c.close()
