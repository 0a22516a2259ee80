"""Where does qb_factor_host's time go beyond the device factorization?  T-sized FP64 A.

    PYTHONPATH=. python tools/e2e_probe.py
"""
import time

import torch

import paper_1503_07157_b200 as qbp
import synth


cfg = synth.CONFIGS["T"]
sig = synth.config_sigma(cfg)
A0 = synth.make_matrix_torch(cfg.m, cfg.n, sig, cfg.seed_matrix, device="cuda", dtype=torch.float64)
m, n, b, q = cfg.m, cfg.n, cfg.b, cfg.q
ctx = qbp.QB(0)
A_h = torch.empty((n, m), dtype=torch.float64, pin_memory=True).t()
A_h.copy_(A0)
g = ctx.factor(A0, cfg.eps, b, q, seed=cfg.seed_omega, copy_out=False)
k = g["k"]
kcap = k + b
Q_h = torch.empty((kcap, m), dtype=torch.float64, pin_memory=True)
B_h = torch.empty((kcap, n), dtype=torch.float64, pin_memory=True)
D = torch.empty_like(A0)


def ev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) / reps * 1e3


print("h2d only        %.1f / %.1f ms" % ev_time(lambda: D.copy_(A_h, non_blocking=True)))
print("factor (device) %.1f / %.1f ms" % ev_time(lambda: ctx.factor(A0, cfg.eps, b, q, seed=cfg.seed_omega,
                                                                    copy_out=False)))
print("factor_host     %.1f / %.1f ms" % ev_time(lambda: qbp.qb_factor_host(
    ctx.ctx, A_h.data_ptr(), m, n, m, cfg.eps, b, q, cfg.seed_omega, 0, Q_h.data_ptr(), m, B_h.data_ptr(), n, kcap)))
print("factor_host, no Q/B copies %.1f / %.1f ms" % ev_time(lambda: qbp.qb_factor_host(
    ctx.ctx, A_h.data_ptr(), m, n, m, cfg.eps, b, q, cfg.seed_omega, 0, Q_h.data_ptr(), m, B_h.data_ptr(), n, 0)))

for kc in (kcap, 0):
    qbp.qb_factor_host(ctx.ctx, A_h.data_ptr(), m, n, m, cfg.eps, b, q, cfg.seed_omega, 0, Q_h.data_ptr(), m,
                       B_h.data_ptr(), n, kc)
    st = qbp.qb_stats(ctx.ctx)
    print("kcap", kc, "block ms", [round(s["ms"], 2) for s in st], "sum", round(sum(s["ms"] for s in st), 1))
