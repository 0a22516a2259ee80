"""qb_factor_host on T with QB_HOST_TIMING=1: host enqueue / wait time per block."""
import torch

import paper_1503_07157_b200 as qbp
import synth

cfg = synth.CONFIGS["T"]
A0 = synth.make_matrix_torch(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix, device="cuda",
                             dtype=torch.float64)
m, n, b, q = cfg.m, cfg.n, cfg.b, cfg.q
ctx = qbp.QB(0)
A_h = torch.empty((n, m), dtype=torch.float64, pin_memory=True).t()
A_h.copy_(A0)
kcap = 2816 + b
Q_h = torch.empty((kcap, m), dtype=torch.float64, pin_memory=True)
B_h = torch.empty((kcap, n), dtype=torch.float64, pin_memory=True)
for kc in (kcap, kcap, 0):
    print("kcap", kc, flush=True)
    qbp.qb_factor_host(ctx.ctx, A_h.data_ptr(), m, n, m, cfg.eps, b, q, cfg.seed_omega, 0, Q_h.data_ptr(), m,
                       B_h.data_ptr(), n, kc)
    torch.cuda.synchronize()
