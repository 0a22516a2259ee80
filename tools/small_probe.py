"""Per-block host enqueue / device timing of a small config (QB_HOST_TIMING=1 prints per block)."""
import sys, time, json
sys.path.insert(0, '.')
import torch, synth, paper_1503_07157_b200 as qbp
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
A = synth.make_matrix_torch(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix)
c = qbp.QB(0)
for i in range(4):
    l0 = c.launches()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = c.factor(A, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega, copy_out=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(json.dumps(dict(cfg=cfg.name, k=g["k"], ms=dt * 1e3, launches=c.launches() - l0,
                          block_ms=[round(s["ms"], 3) for s in g["stats"]][:4])), flush=True)
