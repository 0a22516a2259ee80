"""C4 orthogonality and residual of the FP32 path (for DESIGN R18d).  PYTHONPATH=. python tools/c4_orth.py"""
import torch

import synth
import paper_1503_07157_b200 as qbp

cfg = synth.CONFIGS["C4"]
A = synth.make_matrix_torch(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix, dtype=torch.float32)
c = qbp.QB(0, dtype=qbp.QB_F32)
g = c.factor(A, cfg.eps, cfg.b, cfg.q, cfg.seed_omega)
Q, B = g["Q"].double(), g["B"].double()
k = g["k"]
orth = (Q.T @ Q - torch.eye(k, dtype=torch.float64, device=Q.device)).abs().max().item()
res = torch.linalg.norm(A.double() - Q @ B).item()
print(f"C4 k={k} orth_max={orth:.3e} true_resid={res:.6e} reported={g['resid']:.6e} rel_gap={(g['resid'] - res) / res:.2e}")
