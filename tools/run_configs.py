"""Time every BASELINE config once warm through the public API (evidence table for DESIGN.md).

    python tools/run_configs.py [C1 C2 ...]   ->  one JSON line per config
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_1503_07157_b200 as qbp  # noqa: E402
from bench import falg  # noqa: E402


def run(name, reps=2):
    cfg = synth.CONFIGS[name]
    sig = synth.config_sigma(cfg)
    dt = torch.float32 if cfg.dtype == "f32" else torch.float64
    A0 = synth.make_matrix_torch(cfg.m, cfg.n, sig, cfg.seed_matrix, dtype=dt)
    ctx = qbp.QB(0, dtype=qbp.QB_F32 if cfg.dtype == "f32" else qbp.QB_F64)
    times = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g = ctx.factor(A0, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega, copy_out=False)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = min(times[1:])
    k = g["k"]
    F = falg(cfg.m, cfg.n, k, cfg.b, cfg.q, len(g["stats"]))
    Q, B = g["Q"].double(), g["B"].double()
    orth = (Q.T @ Q - torch.eye(k, dtype=torch.float64, device="cuda")).abs().max().item() if k else 0.0
    true = torch.linalg.norm(A0.double() - Q @ B).item() if cfg.m * cfg.n <= 4e8 else None
    out = dict(config=name, m=cfg.m, n=cfg.n, dtype=cfg.dtype, b=cfg.b, q=cfg.q, eps=cfg.eps, k=k,
               k_eps=synth.eps_rank(sig, cfg.eps), status=g["status"], ms=ms, gflops=F / ms * 1e-6,
               frac_fp64_peak=F / ms * 1e-9 / 37.186, orth_max=orth, resid=g["resid"], true_resid=true)
    ctx.close()
    del A0
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "T", "T1", "C5"]
    for nm in names:
        print(json.dumps(run(nm)), flush=True)
