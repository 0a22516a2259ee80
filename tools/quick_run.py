"""Quick timing of one config through the public API (development helper, not the bench)."""
import sys
import time

import torch

import synth
import paper_1503_07157_b200 as qbp

name = sys.argv[1] if len(sys.argv) > 1 else "T"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = synth.CONFIGS[name]
sig = synth.config_sigma(cfg)
t = time.time()
dt = torch.float32 if cfg.dtype == "f32" else torch.float64
A0 = synth.make_matrix_torch(cfg.m, cfg.n, sig, cfg.seed_matrix, dtype=dt)
torch.cuda.synchronize()
print(f"gen {time.time() - t:.2f}s", flush=True)
ctx = qbp.QB(0, dtype=qbp.QB_F32 if cfg.dtype == "f32" else qbp.QB_F64)
A = torch.empty_like(A0)
for r in range(reps):
    A.copy_(A0)
    torch.cuda.synchronize()
    t = time.time()
    g = ctx.factor(A, cfg.eps, cfg.b, cfg.q, cfg.seed_omega, overwrite=True, copy_out=False)
    torch.cuda.synchronize()
    dt = time.time() - t
    k = g["k"]
    m, n, b, q = cfg.m, cfg.n, cfg.b, cfg.q
    s = len(g["stats"])
    F = (3 + 2 * q) * 2 * m * n * k + 2 * m * k * (k - b) + s * ((2 + q) * 4 * m * b * b + q * 4 * n * b * b)
    print(f"{name} rep{r}: {dt * 1e3:.1f} ms k={k} status={g['status']} resid={g['resid']:.3e} "
          f"GF/s={F / dt * 1e-9:.0f} frac37.2={F / dt / 37.2e12:.3f} launches={ctx.launches()}", flush=True)
    print("  block ms:", [round(x["ms"], 2) for x in g["stats"]], "fallbacks", sum(x["fallback"] for x in g["stats"]))
    st = g["stats"]
    sk = sum(x["ms_sketch"] for x in st); bm = sum(x["ms_bmat"] for x in st); dn = sum(x["ms_down"] for x in st)
    tot = sum(x["ms"] for x in st)
    print(f"  phases: sketch {sk:.1f} ms, B {bm:.1f} ms, downdate {dn:.1f} ms, rest (orth/reproj/power/sync) "
          f"{tot - sk - bm - dn:.1f} ms of {tot:.1f} ms")
