#!/usr/bin/env python
"""bench.py — benchmark of the QB hot path, driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config T] [--impl ours|reference]

A "step" is one full adaptive factorization (all rows of SURVEY.md §8(a): Ω, sketch, orth,
re-projection, B, downdate, stop test) of the N=1 workload "T" — the north_star target:
A = U diag(σ) V^* 20000 x 20000 FP64, σ_j = e^(-j/150), eps = 1e-6, b = 256, q = 0 —
through the C ABI with A resident in HBM (``value``), and through the host-buffer entry
point with the H2D copy of A and the D2H copy of Q, B inside the timed region (``e2e``).
The metric is BASELINE.json's: FP64 GFLOP/s of the algorithmic work F_alg (DESIGN.md §8,
PAPER.md:902 cost model with C_mm = 2) and seconds-to-eps, as a fraction of the FP64 peak.

Multi-GPU (torchrun, N > 1): the column-sharded path — every rank owns a
column block of A, Y_i and the norm scalars are summed with NCCL, orth is replicated, B_i and
the downdate stay local.  Default "weak" scaling: every rank holds a 20000 x 20000 block of
the 20000 x 20000N matrix with the T spectrum (synth.make_shard_torch), so per-GPU work is
fixed; ``--strong`` shards the one 20000 x 20000 T matrix instead.  The time is the max over
ranks; ``value`` is the algorithmic work of the whole (global) factorization per second.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 seconds-to-eps and GFLOP/s (frac of B200 FP64 tensor peak)"
FP64_PEAK_FALLBACK = 37.2  # TFLOP/s: 148 SM x 128 flop/clk x 1.965 GHz (derived)


def falg(m, n, k, b, q, s):
    """Algorithmic FP64 flops of one factorization: (3+2q) GEMM passes of
    2mnw per block, the re-projection 2 m k (k - b), and Householder-equivalent orth."""
    return ((3 + 2 * q) * 2.0 * m * n * k + 2.0 * m * k * max(k - b, 0)
            + s * ((2 + q) * 4.0 * m * b * b + q * 4.0 * n * b * b))


def fp64_peak():
    p = os.path.join(ROOT, "profiles", "MEASURED_FP64.json")
    try:
        d = json.load(open(p))
        return float(d["dmma_peak_tflops"]), "measured DMMA microbenchmark (profiles/MEASURED_FP64.json)", \
            float(d.get("cublas_dgemm_8192_tflops", 0.0)) or None
    except Exception:
        return FP64_PEAK_FALLBACK, "derived 148 SM x 128 flop/clk x 1.965 GHz", None


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9 or not parts[0].isdigit() or int(parts[0]) != self.index:
                continue
            rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "samples": len(rows), "reasons": sorted(reasons)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_A(cfg, device):
    import torch
    import synth
    dt = torch.float32 if cfg.dtype == "f32" else torch.float64
    return synth.make_matrix_torch(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix, device=device, dtype=dt)


def hbm_peak():
    """Measured copy bandwidth (driver-written MEASURED_PEAKS.json), else the guide's figure."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 7700.0, "B200_PROFILING.md nominal HBM3e 7.7 TB/s"


def oracle_sample(A_np, cfg, blocks):
    """Time the oracle (as it stands) on the first `blocks` blocks of the workload."""
    from oracle import qb as oqb
    t0 = time.perf_counter()
    r = oqb.randqb_pb(A_np, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega, kmax=blocks * cfg.b)
    dt = time.perf_counter() - t0
    F = falg(cfg.m, cfg.n, r.k, cfg.b, cfg.q, len(r.hist))
    return F, dt, r.k


def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        info = [x for x in threadpool_info() if x.get("user_api") == "blas"]
        if info:
            return int(info[0]["num_threads"])
    except Exception:
        pass
    return os.cpu_count()


def workload_desc(cfg):
    return (f"{cfg.name}: A = U diag(sigma) V^T {cfg.m}x{cfg.n} {cfg.dtype.upper()}, sigma_j = {cfg.spectrum}, "
            f"eps = {cfg.eps:g}, b = {cfg.b}, q = {cfg.q}")


def run_reference(args, cfg):
    """--impl reference: the CPU oracle timed on the host cores, bounded sample per step."""
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    import numpy as np
    import torch
    dev = f"cuda:{local}" if torch.cuda.is_available() else "cpu"
    A_np = np.asfortranarray(make_A(cfg, dev).cpu().numpy()) if dev != "cpu" else None
    if A_np is None:
        import synth
        A_np = synth.make_matrix_np(cfg.m, cfg.n, synth.config_sigma(cfg), cfg.seed_matrix)
    blocks = args.cpu_sample_blocks
    for _ in range(args.warmup):
        oracle_sample(A_np, cfg, blocks)
    Fs, ts = 0.0, 0.0
    k = 0
    for _ in range(args.steps):
        F, dt, k = oracle_sample(A_np, cfg, blocks)
        Fs += F
        ts += dt
    gf = Fs / ts * 1e-9
    cores = oracle_threads()
    sample = f"first {blocks} block(s) of the workload (kmax = {blocks * cfg.b}, k = {k}) per step"
    line = {"impl": "reference", "metric": METRIC, "value": gf, "unit": "GFLOP/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ts / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "l2": "inputs larger than L2 (A is 3.2 GB)"},
            "cpu_baseline": {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": gf, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1503_07157_b200 as qbp
    import synth

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dspec = None
    sig = synth.config_sigma(cfg)
    f32 = cfg.dtype == "f32"
    tdt = torch.float32 if f32 else torch.float64
    es = 4 if f32 else 8
    # tall-skinny workloads shard rows (NEXT-2), square ones columns; --shard overrides
    rows = (args.shard == "rows") or (args.shard == "auto" and cfg.m >= 8 * cfg.n)
    m_global, m_local = cfg.m, cfg.m
    if ws > 1:
        from paper_1503_07157_b200.dist import dist_spec, dist_spec_rows
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        if rows:
            m_global = cfg.m if args.strong else cfg.m * ws
            dspec = dist_spec_rows(m_global)
        else:
            n_global = cfg.n if args.strong else cfg.n * ws
            dspec = dist_spec(n_global)
    dev = torch.device(f"cuda:{local}")
    stream = torch.cuda.current_stream(dev)
    if dspec is None:
        A0 = make_A(cfg, dev)
        n_global, n_local = cfg.n, cfg.n
    elif rows:
        n_global, n_local = cfg.n, cfg.n
        if args.strong:
            Af = make_A(cfg, dev)
            off, m_local = dspec["row_offset"], dspec["m_local"]
            A0 = Af[off:off + m_local].t().contiguous().t()
            del Af
        else:
            m_local = cfg.m
            dspec["row_offset"], dspec["m_local"] = rank * m_local, m_local
            A0 = synth.make_row_shard_torch(m_local, cfg.n, sig, cfg.seed_matrix, rank, ws, device=dev, dtype=tdt)
    elif args.strong:
        Af = make_A(cfg, dev)
        off, n_local = dspec["col_offset"], dspec["n_local"]
        A0 = Af.t()[off:off + n_local].contiguous().t()
        del Af
        n_global = cfg.n
    else:
        n_local = cfg.n
        n_global = cfg.n * ws
        dspec["col_offset"], dspec["n_local"] = rank * n_local, n_local
        A0 = synth.make_shard_torch(cfg.m, n_local, sig, cfg.seed_matrix, rank, ws, device=dev, dtype=tdt)
    torch.cuda.synchronize()
    ctx = qbp.QB(local, dtype=qbp.QB_F32 if f32 else qbp.QB_F64, stream=ctypes_stream(stream), dist=dspec)
    m, b, q = m_local, cfg.b, cfg.q

    def step():
        return ctx.factor(A0, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega, copy_out=False)

    g = None
    for _ in range(args.warmup):
        g = step()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = ctx.launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        g = step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launches() - l0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    k, stats = g["k"], g["stats"]
    F = falg(m_global, n_global, k, b, q, len(stats))
    value = F / (ms * 1e-3) * 1e-9
    peak, peak_src, cublas = fp64_peak()

    # roofline of the dominant kernel: the downdate GEMM A -= Q_i B_i (fused norm epilogue)
    full = [s for s in stats if s["w"] == b] or stats
    t_down = statistics.mean(s["ms_down"] for s in full) * 1e-3
    if not f32:
        achieved = 2.0 * m * n_local * b / t_down * 1e-12
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_summary_r01d.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("downdate_dram_bytes_per_launch")
            except Exception:
                traffic = None
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "kernel": "gemm_f64_kernel<NN,64,SUB_COL> (A -= Q_i B_i, fused ||A||_F^2)",
                    "peak_source": peak_src,
                    "algorithmic_per_launch": f"2*m*n_local*b = {2.0 * m * n_local * b:.4g} flop",
                    "share_of_step": sum(s["ms_down"] for s in stats) / ms}
    else:  # FP32: the 3xTF32 subtract-update streams A in and out of HBM (K = b is short)
        hbm, hbm_src = hbm_peak()
        achieved = 2.0 * m * n_local * 4 / t_down * 1e-9
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_summary_r01h_tf32.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("downdate_dram_bytes_per_launch")
            except Exception:
                traffic = None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": traffic,
                    "kernel": "gemm_tf32_sub_ares_kernel<128> (A -= Q_i B_i, 3xTF32, A rows resident in TMEM, "
                              "fused ||A||_F^2)",
                    "peak_source": hbm_src,
                    "algorithmic_per_launch": f"2*m*n_local*4 = {2.0 * m * n_local * 4:.4g} bytes (A read + write)",
                    "share_of_step": sum(s["ms_down"] for s in stats) / ms}

    # end to end through the host-buffer entry point: H2D of A, D2H of Q and B per step
    e2e = None
    if not args.no_e2e:
        A_h = torch.empty((n_local, m), dtype=tdt, pin_memory=True).t()   # column-major host A
        A_h.copy_(A0)
        kcap = k + b
        Q_h = torch.empty((kcap, m), dtype=tdt, pin_memory=True)
        B_h = torch.empty((kcap, n_local), dtype=tdt, pin_memory=True)
        res = qbp.qb_factor_host(ctx.ctx, A_h.data_ptr(), m, n_local, m, cfg.eps, b, q, cfg.seed_omega, 0,
                                 Q_h.data_ptr(), m, B_h.data_ptr(), n_local, kcap)
        torch.cuda.synchronize()
        esteps = max(1, min(args.steps, 3))
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(esteps):
            res = qbp.qb_factor_host(ctx.ctx, A_h.data_ptr(), m, n_local, m, cfg.eps, b, q, cfg.seed_omega, 0,
                                     Q_h.data_ptr(), m, B_h.data_ptr(), n_local, kcap)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / esteps * 1e3
        ems = max(e0.elapsed_time(e1) / esteps, wall)
        if ws > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        ke = res["k"]
        e2e = {"value": falg(m_global, n_global, ke, b, q, -(-ke // b)) / (ems * 1e-3) * 1e-9, "unit": "GFLOP/s",
               "ms_per_step": ems, "h2d_bytes_per_step": ws * m * n_local * es,
               "d2h_bytes_per_step": ws * ke * (m + n_local) * es + 16,
               "entry_point": "qb_factor_host (pinned host A, Q, B; every rank its shard)"}
        del A_h, Q_h, B_h

    # the NEXT rows timed once each after the main measurement (warm, CUDA events, not in `value`):
    # QB -> SVD (rqb_svd) and QB -> pivoted QR (qb_pivoted_qr) of the last factorization, and the
    # fixed-rank randQB at l = k (one wide GEMM per product instead of s narrow ones)
    post = None
    if ws == 1 and not args.no_post:
        post = {}
        for name, fn in (("rqb_svd", lambda: ctx.svd(copy_out=False)),
                         ("pivoted_qr", lambda: ctx.pivoted_qr(copy_out=False)),
                         ("fixed_rank_randQB_l_eq_k", lambda: ctx.fixed_rank(A0, k, 0, seed=cfg.seed_omega,
                                                                            want_resid=False, copy_out=False))):
            fn()  # warm (svd and pivoted QR read the last factorization; fixed_rank runs last)
            torch.cuda.synchronize()
            p0 = torch.cuda.Event(enable_timing=True)
            p1 = torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            fn()
            p1.record(stream)
            torch.cuda.synchronize()
            post[name + "_ms"] = p0.elapsed_time(p1)
        post["k"] = k

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        A_np = np.asfortranarray(A0.cpu().numpy())
        Fc, tc, kc = oracle_sample(A_np, cfg, args.cpu_sample_blocks)
        cpu = {"value": Fc / tc * 1e-9, "unit": "GFLOP/s", "cores": oracle_threads(), "kind": "oracle",
               "sample": f"first {args.cpu_sample_blocks} block(s) of the workload (kmax = "
                         f"{args.cpu_sample_blocks * b}), {tc:.1f} s of CPU work", "seconds": tc}
        del A_np

    if rank == 0:
        scaling = "strong" if (ws > 1 and args.strong) else "weak"
        par = "single" if ws == 1 else (
            f"row-sharded x{ws} (NCCL allreduce of Grams, W, Z, B_i, norms)" if rows else
            f"column-sharded x{ws} (NCCL allreduce of Y_i, Gram, norms)")
        line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
                "config": {"workload": workload_desc(cfg) + ("" if ws == 1 else
                           f"; {'one matrix sharded' if args.strong else 'weak: %d x %d global' % (m_global, n_global)}"),
                           "m": m_global, "n": n_global, "m_per_gpu": m, "n_per_gpu": n_local, "b": b, "q": q,
                           "eps": cfg.eps, "k": k, "blocks": len(stats), "parallelism": par,
                           "l2": f"inputs larger than L2 (A is {m * n_local * es / 1e9:.1f} GB per GPU; every step "
                                 "reads it >= 3 times)"},
                "seconds_to_eps": ms * 1e-3,
                "frac_fp64_peak": None if f32 else value / ws / (peak * 1e3),
                "frac_cublas_dgemm": (value / ws / (cublas * 1e3)) if (cublas and not f32) else None,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "post": post,
                "clocks": clk}
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def ctypes_stream(stream):
    import ctypes
    return ctypes.c_void_p(stream.cuda_stream or 1)   # 0 (legacy default) -> cudaStreamLegacy


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="T")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-blocks", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-post", action="store_true", help="skip timing rqb_svd / pivoted QR / fixed-rank")
    ap.add_argument("--strong", action="store_true", help="N > 1: shard one matrix (strong scaling)")
    ap.add_argument("--shard", default="auto", choices=["auto", "cols", "rows"],
                    help="N > 1: shard columns (square A) or rows (tall-skinny A, NEXT-2); auto picks rows "
                         "when m >= 8 n")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    import synth
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
