"""qb_pivoted_qr on a config after a factorization: warm timing (CUDA events), for launch lists too.

    PYTHONPATH=. python tools/qrcp_once.py [C3|T]
"""
import sys

import torch

import paper_1503_07157_b200 as qbp
import synth

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
A = synth.make_matrix_torch(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix, dtype=torch.float64)
c = qbp.QB(0)
g = c.factor(A, cfg.eps, cfg.b, cfg.q, cfg.seed_omega, copy_out=False)
torch.cuda.synchronize()
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = c.pivoted_qr(copy_out=False)
    e1.record()
    torch.cuda.synchronize()
    print(f"k {g['k']} pivoted_qr {e0.elapsed_time(e1):.1f} ms", flush=True)
