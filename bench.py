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

Multi-GPU (N > 1): one process per GPU over NCCL.  Under torchrun the ranks
come from the environment; ``--gpus N`` without torchrun relaunches itself under
torch.distributed.run, and fails loudly when fewer than N GPUs are visible.  Default is
STRONG scaling: one matrix is sharded (columns for square A, rows for tall-skinny A, NEXT-2),
so the N = 1 point is the single-GPU measurement; ``--weak`` gives every rank its own
20000 x 20000 block of a 20000 x 20000N matrix instead.  The time is the max over ranks;
``value`` is the algorithmic work of the whole factorization per second.

Beside the main workload the line carries ``configs``: one record per other BASELINE config
(C1, C2, C3, C4 FP32, C5 and T1 = T with q = 1 at N = 1; the sharded C3, C4, C5, T1 at N > 1),
each timed the same way (device-resident A, CUDA events, W warm-up steps, max over ranks).
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


def tf32x3_peak():
    """3xTF32 tensor ceiling for the FP32 path: the measured dense BF16 rate x the nominal
    TF32/BF16 ratio (1/2), / 3 MMAs per FP32-equivalent product."""
    try:
        bf16 = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
        return bf16 / 2 / 3, "MEASURED_PEAKS.json bf16 x 1/2 (TF32) / 3 (3xTF32)"
    except Exception:
        return 2250.0 / 2 / 3, "nominal 2.25 PF bf16 x 1/2 / 3"


def bytes_alg(m, n, k, b, q, s, es):
    """Algorithmic HBM bytes: (3+2q) passes over A per block + the re-projection's
    reads of Q̄ (sum_i 2 m ell_{i-1} es)."""
    ells = [min(i * b, k) for i in range(s)]
    return s * (3 + 2 * q) * m * n * es + sum(2 * m * l * es for l in ells)


def shard_inputs(cfg, ws, rank, local, weak, shard):
    """This rank's block of the workload's A (device-resident, column-major) and its descriptor.
    rows: tall-skinny A sharded by rows (NEXT-2), else columns.  Strong scaling (default) slices
    one matrix; weak scaling builds an m x n block of an (m x nP) or (mP x n) matrix with the
    same spectrum (synth.make_shard_torch / make_row_shard_torch)."""
    import torch
    import synth
    sig = synth.config_sigma(cfg)
    tdt = torch.float32 if cfg.dtype == "f32" else torch.float64
    dev = torch.device(f"cuda:{local}")
    rows = (shard == "rows") or (shard == "auto" and cfg.m >= 8 * cfg.n)
    out = dict(rows=rows, dspec=None, m_global=cfg.m, n_global=cfg.n, m_local=cfg.m, n_local=cfg.n)
    if ws == 1:
        out["A0"] = make_A(cfg, dev)
        return out
    from paper_1503_07157_b200.dist import dist_spec, dist_spec_rows
    if rows:
        out["m_global"] = cfg.m * ws if weak else cfg.m
        d = dist_spec_rows(out["m_global"])
        if weak:
            d["row_offset"], d["m_local"] = rank * cfg.m, cfg.m
            out["A0"] = synth.make_row_shard_torch(cfg.m, cfg.n, sig, cfg.seed_matrix, rank, ws, device=dev, dtype=tdt)
        else:
            Af = make_A(cfg, dev)
            off, ml = d["row_offset"], d["m_local"]
            out["A0"] = Af[off:off + ml].t().contiguous().t()
            del Af
        out["m_local"] = d["m_local"]
    else:
        out["n_global"] = cfg.n * ws if weak else cfg.n
        d = dist_spec(out["n_global"])
        if weak:
            d["col_offset"], d["n_local"] = rank * cfg.n, cfg.n
            out["A0"] = synth.make_shard_torch(cfg.m, cfg.n, sig, cfg.seed_matrix, rank, ws, device=dev, dtype=tdt)
        else:
            Af = make_A(cfg, dev)
            off, nl = d["col_offset"], d["n_local"]
            out["A0"] = Af.t()[off:off + nl].contiguous().t()
            del Af
        out["n_local"] = d["n_local"]
    out["dspec"] = d
    torch.cuda.synchronize()
    return out


def timed_steps(step, steps, warmup, stream, ws, dev, flush=None):
    """W untimed warm-up steps, then K steps timed with CUDA events on the library's stream,
    bracketed by a barrier + synchronize; max over ranks.  flush: an L2 flush run between
    timed steps outside the events (inputs smaller than L2)."""
    import torch
    import torch.distributed as dist
    g = None
    for _ in range(warmup):
        g = step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total = 0.0
    if flush is None:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            g = step()
        e1.record(stream)
        torch.cuda.synchronize()
        total = e0.elapsed_time(e1)
    else:
        for _ in range(steps):
            flush()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g = step()
            e1.record(stream)
            torch.cuda.synchronize()
            total += e0.elapsed_time(e1)
    ms = total / steps
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    return ms, g


def replicated_share(stats, ms):
    """rho of SURVEY §8(e): the share of a step spent in the work column sharding replicates on every
    rank — CholeskyQR of the m-row panels, the re-projection, and (upper bound) the power steps'
    CholeskyQR of Z, whose Gram and products are in fact sharded — from qb_stats' phase spans."""
    rep = sum(s["ms_orth"] + s["ms_orth_z"] + s["ms_reproj"] for s in stats)
    return {"rho": rep / ms, "orth_ms": sum(s["ms_orth"] for s in stats),
            "orth_z_ms": sum(s["ms_orth_z"] for s in stats), "reproj_ms": sum(s["ms_reproj"] for s in stats),
            "power_gemm_ms": sum(s["ms_power"] for s in stats)}


RECORD_STEPS = {"C1": 20, "C2": 20, "C3": 5, "C4": 5, "C5": 2, "T1": 3, "T": 5}


def run_record(name, args, ws, rank, local):
    """One BASELINE config timed like the main workload (device-resident A, CUDA events,
    >= 3 warm-up steps, max over ranks), strong-sharded over the N ranks."""
    import torch
    import paper_1503_07157_b200 as qbp
    import synth
    cfg = synth.CONFIGS[name]
    f32 = cfg.dtype == "f32"
    es = 4 if f32 else 8
    inp = shard_inputs(cfg, ws, rank, local, False, args.shard)
    dev = torch.device(f"cuda:{local}")
    stream = torch.cuda.current_stream(dev)
    ctx = qbp.QB(local, dtype=qbp.QB_F32 if f32 else qbp.QB_F64, stream=ctypes_stream(stream), dist=inp["dspec"])
    A0 = inp["A0"]
    flush = None
    l2_note = f"inputs larger than L2 (A is {A0.numel() * es / 1e9:.2f} GB per GPU)"
    if A0.numel() * es < 512e6:   # A not far above the 126 MB L2: flush it between timed steps
        junk = torch.empty(int(256e6) // 4, dtype=torch.float32, device=dev)
        flush = lambda: junk.fill_(1.0)  # noqa: E731
        l2_note = "L2 flushed between timed steps (256 MB write)"
    steps = RECORD_STEPS.get(name, 3)
    ms, g = timed_steps(lambda: ctx.factor(A0, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega, copy_out=False),
                        steps, max(3, args.warmup if name in ("C1", "C2") else 3), stream, ws, dev, flush)
    k, st = g["k"], g["stats"]
    F = falg(inp["m_global"], inp["n_global"], k, cfg.b, cfg.q, len(st))
    rec = {"ms_per_step": ms, "value": F / (ms * 1e-3) * 1e-9, "unit": "GFLOP/s", "seconds_to_eps": ms * 1e-3,
           "k": k, "blocks": len(st), "status": g["status"], "m": inp["m_global"], "n": inp["n_global"],
           "b": cfg.b, "q": cfg.q, "eps": cfg.eps, "dtype": cfg.dtype, "steps": steps, "warmup": 3, "n_gpus": ws,
           "sharding": "single" if ws == 1 else ("rows" if inp["rows"] else "cols"), "l2": l2_note}
    rec["replicated_share"] = replicated_share(st, ms)
    if f32:
        tf, tf_src = tf32x3_peak()
        hbm, _ = hbm_peak()
        t_flop = F / (tf * 1e12)
        t_hbm = bytes_alg(inp["m_global"], inp["n_global"], k, cfg.b, cfg.q, len(st), es) / (hbm * 1e9)
        rec["roofline"] = {"bound": "tensor" if t_flop >= t_hbm else "hbm", "t_roof_ms": max(t_flop, t_hbm) * 1e3 / ws,
                           "t_flop_ms": t_flop * 1e3 / ws, "t_hbm_ms": t_hbm * 1e3 / ws,
                           "frac": max(t_flop, t_hbm) * 1e3 / ws / ms, "peak_3xtf32_tflops": tf, "peak_source": tf_src}
    else:
        peak, _, _ = fp64_peak()
        rec["frac_fp64_peak"] = rec["value"] / ws / (peak * 1e3)
    ctx.close()
    del A0, inp
    torch.cuda.empty_cache()
    return rec


def latest_profile(pattern_key, names):
    """The newest committed ncu summary among `names` (profiles/) carrying `pattern_key`."""
    for nm in names:
        pth = os.path.join(ROOT, "profiles", nm)
        if os.path.exists(pth):
            try:
                d = json.load(open(pth))
                if d.get(pattern_key) is not None:
                    return d[pattern_key], nm
            except Exception:
                pass
    return None, None


def run_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1503_07157_b200 as qbp

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    f32 = cfg.dtype == "f32"
    tdt = torch.float32 if f32 else torch.float64
    es = 4 if f32 else 8
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    weak = ws > 1 and args.weak
    inp = shard_inputs(cfg, ws, rank, local, weak, args.shard)
    A0, dspec, rows = inp["A0"], inp["dspec"], inp["rows"]
    m_global, n_global, m, n_local = inp["m_global"], inp["n_global"], inp["m_local"], inp["n_local"]
    dev = torch.device(f"cuda:{local}")
    stream = torch.cuda.current_stream(dev)
    ctx = qbp.QB(local, dtype=qbp.QB_F32 if f32 else qbp.QB_F64, stream=ctypes_stream(stream), dist=dspec)
    b, q = cfg.b, cfg.q

    def step():
        return ctx.factor(A0, cfg.eps, cfg.b, cfg.q, seed=cfg.seed_omega, copy_out=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    l0 = ctx.launches()
    ms, g = timed_steps(step, args.steps, 0, stream, ws, dev)
    launches = ctx.launches() - l0
    clk = clocks.stop()
    k, stats = g["k"], g["stats"]
    F = falg(m_global, n_global, k, b, q, len(stats))
    value = F / (ms * 1e-3) * 1e-9
    peak, peak_src, cublas = fp64_peak()

    # roofline of the dominant kernel: the downdate GEMM A -= Q_i B_i (fused norm epilogue)
    full = [s for s in stats if s["w"] == b] or stats
    t_down = statistics.mean(s["ms_down"] for s in full) * 1e-3
    if not f32:
        achieved = 2.0 * m * n_local * b / t_down * 1e-12
        traffic, tsrc = latest_profile("downdate_dram_bytes_per_launch",
                                       ["ncu_summary_r02_down64.json", "ncu_summary_r01k_down64.json"])
        alg_bytes = 2.0 * m * n_local * 8
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "traffic_over_algorithmic_bytes": (traffic / alg_bytes) if traffic else None,
                    "traffic_source": tsrc,
                    "kernel": "gemm_f64_kernel<NN,64,SUB_COL> (A -= Q_i B_i, fused ||A||_F^2)",
                    "peak_source": peak_src,
                    "algorithmic_per_launch": f"2*m*n_local*b = {2.0 * m * n_local * b:.4g} flop "
                                              f"(A read + write = {alg_bytes:.4g} bytes)",
                    "share_of_step": sum(s["ms_down"] for s in stats) / ms}
    else:  # FP32: the 3xTF32 subtract-update streams A in and out of HBM (K = b is short)
        hbm, hbm_src = hbm_peak()
        achieved = 2.0 * m * n_local * 4 / t_down * 1e-9
        traffic, tsrc = latest_profile("downdate_dram_bytes_per_launch", ["ncu_summary_r01h_tf32.json"])
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": traffic, "traffic_source": tsrc,
                    "traffic_over_algorithmic_bytes": (traffic / (2.0 * m * n_local * 4)) if traffic else None,
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

        def estep():
            return qbp.qb_factor_host(ctx.ctx, A_h.data_ptr(), m, n_local, m, cfg.eps, b, q, cfg.seed_omega, 0,
                                      Q_h.data_ptr(), m, B_h.data_ptr(), n_local, kcap)
        esteps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        ems, res = timed_steps(estep, esteps, 1, stream, ws, dev)
        wall = (time.perf_counter() - t0) / (esteps + 1) * 1e3
        ems = max(ems, wall if ws == 1 else 0.0)
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
        step()  # the factorization the post-processing converts
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
    ctx.close()
    del A0, inp
    torch.cuda.empty_cache()

    # the other BASELINE configs, each its own record (strong-sharded over the N ranks)
    names = args.records
    if names == "auto":
        names = "C1,C2,C3,C4,C5,T1" if ws == 1 else "C3,C4,C5,T1"
    records = {}
    for nm in [x for x in names.split(",") if x and x != "none" and x != cfg.name]:
        try:
            records[nm] = run_record(nm, args, ws, rank, local)
        except Exception as e:  # noqa: BLE001 - a failing record is reported, not fatal
            records[nm] = {"error": f"{type(e).__name__}: {e}"}

    if rank == 0:
        scaling = "weak" if weak else "strong"
        par = "single" if ws == 1 else (
            f"row-sharded x{ws} (NCCL allreduce of Grams, W, Z, B_i, norms)" if rows else
            f"column-sharded x{ws} (NCCL allreduce of Y_i, Gram, norms)")
        line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
                "config": {"workload": workload_desc(cfg) + ("" if ws == 1 else
                           ("; one matrix sharded" if not weak else f"; weak: {m_global} x {n_global} global")),
                           "m": m_global, "n": n_global, "m_per_gpu": m, "n_per_gpu": n_local, "b": b, "q": q,
                           "eps": cfg.eps, "k": k, "blocks": len(stats), "parallelism": par,
                           "l2": f"inputs larger than L2 (A is {m * n_local * es / 1e9:.1f} GB per GPU; every step "
                                 "reads it >= 3 times)"},
                "seconds_to_eps": ms * 1e-3,
                "frac_fp64_peak": None if f32 else value / ws / (peak * 1e3),
                "frac_cublas_dgemm": (value / ws / (cublas * 1e3)) if (cublas and not f32) else None,
                "replicated_share": replicated_share(stats, ms),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "post": post,
                "configs": records, "clocks": clk}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def relaunch_under_torchrun(n):
    """--gpus N without torchrun: start N ranks with torch.distributed.run (127.0.0.1), or fail
    loudly when fewer than N GPUs are visible (never a silent single-rank run)."""
    import socket
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:  # pragma: no cover
        have = 0
    if have < n:
        sys.stderr.write(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}\n")
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
    ap.add_argument("--strong", action="store_true", help="N > 1: shard one matrix (strong scaling; the default)")
    ap.add_argument("--weak", action="store_true", help="N > 1: every rank its own 20000^2 block (weak scaling)")
    ap.add_argument("--records", default="auto",
                    help="comma-separated extra configs timed into the line's `configs` ('none' to skip); "
                         "auto = C1,C2,C3,C4,C5,T1 at N = 1 and C3,C4,C5,T1 at N > 1")
    ap.add_argument("--shard", default="auto", choices=["auto", "cols", "rows"],
                    help="N > 1: shard columns (square A) or rows (tall-skinny A, NEXT-2); auto picks rows "
                         "when m >= 8 n")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if ws == 0 and args.gpus > 1:
        return relaunch_under_torchrun(args.gpus)
    if ws > 0 and ws != args.gpus and not (ws == 1 and args.gpus <= 1):
        sys.stderr.write(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}\n")
        return 2
    import synth
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
