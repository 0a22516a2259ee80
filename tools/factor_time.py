"""Warm qb_factor timing (CUDA events, A not overwritten: the library's working copy included).

    PYTHONPATH=. python tools/factor_time.py [T|C4|...] [reps]
"""
import sys

import torch

import paper_1503_07157_b200 as qbp
import synth

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "T"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dt = torch.float32 if cfg.dtype == "f32" else torch.float64
A = synth.make_matrix_torch(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix, dtype=dt)
c = qbp.QB(0, dtype=qbp.QB_F32 if cfg.dtype == "f32" else qbp.QB_F64)
for _ in range(2):
    g = c.factor(A, cfg.eps, cfg.b, cfg.q, cfg.seed_omega, copy_out=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    g = c.factor(A, cfg.eps, cfg.b, cfg.q, cfg.seed_omega, copy_out=False)
e1.record()
torch.cuda.synchronize()
print(f"{qbp.LIB_PATH.split('/')[-1]} {sys.argv[1] if len(sys.argv) > 1 else 'T'} k={g['k']} "
      f"{e0.elapsed_time(e1) / reps:.2f} ms  r0^2-derived resid {g['resid']:.6e}", flush=True)
