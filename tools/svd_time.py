import sys, time, json
sys.path.insert(0, '.')
import torch, synth, paper_1503_07157_b200 as qbp
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "T"]
A = synth.make_matrix_torch(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix,
                            dtype=torch.float32 if cfg.dtype == "f32" else torch.float64)
c = qbp.QB(0, dtype=qbp.QB_F32 if cfg.dtype == "f32" else qbp.QB_F64)
g = c.factor(A, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega, copy_out=False)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s = c.svd(copy_out=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(json.dumps(dict(cfg=cfg.name, k=g["k"], ms=dt * 1e3, sweeps=qbp.qb_svd_sweeps(c.ctx))), flush=True)
S = s["S"].double()
print("S head", S[:3].tolist(), "tail", S[-3:].tolist())
