"""One warm factorization of a config (for ncu launch lists).  PYTHONPATH=. python tools/factor_once.py C4"""
import sys

import torch

import synth
import paper_1503_07157_b200 as qbp

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = synth.CONFIGS[name]
dt = torch.float32 if cfg.dtype == "f32" else torch.float64
A = synth.make_matrix_torch(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix, dtype=dt)
c = qbp.QB(0, dtype=qbp.QB_F32 if cfg.dtype == "f32" else qbp.QB_F64)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    g = c.factor(A, cfg.eps, cfg.b, cfg.q, cfg.seed_omega, copy_out=False)
torch.cuda.synchronize()
print(name, "k", g["k"], "launches", c.launches())
