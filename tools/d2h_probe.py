"""Does work enqueued on a blocking stream right after a large D2H on a non-blocking stream
wait for that copy?  (qb_factor_host: block i's Q_i / B_i copies, then block i+1's kernels)"""
import ctypes
import time

import torch

import paper_1503_07157_b200 as qbp  # noqa: F401  (loads the same libcudart)

rt = ctypes.CDLL("libcudart.so.12")
m, w = 20000, 256
src = torch.randn(2 * w, m, dtype=torch.float64, device="cuda")
Q_h = torch.empty((3072, m), dtype=torch.float64, pin_memory=True)
cs = ctypes.c_void_p()
rt.cudaStreamCreateWithFlags(ctypes.byref(cs), 1)  # non-blocking copy stream
ms_ = ctypes.c_void_p()
rt.cudaStreamCreateWithFlags(ctypes.byref(ms_), 0)  # blocking main stream
main = torch.cuda.ExternalStream(ms_.value)
x = torch.randn(1024, device="cuda")
for mode, timing in (("2d", False), ("2d", True), ("none", True)):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if mode == "2d":
            rt.cudaMemcpy2DAsync(ctypes.c_void_p(Q_h.data_ptr()), ctypes.c_size_t(m * 8), ctypes.c_void_p(src.data_ptr()),
                                 ctypes.c_size_t(m * 8), ctypes.c_size_t(m * 8), ctypes.c_size_t(2 * w), 2, cs)
        elif mode == "1d":
            rt.cudaMemcpyAsync(ctypes.c_void_p(Q_h.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                               ctypes.c_size_t(2 * w * m * 8), 2, cs)
        e = torch.cuda.Event(enable_timing=timing)
        with torch.cuda.stream(main):
            x.add_(1.0)
            e.record(main)
        e.synchronize()
        t1 = time.perf_counter()
        rt.cudaStreamSynchronize(cs)
        t2 = time.perf_counter()
        print(f"{mode} timing={timing}: main-stream kernel done after {1e3 * (t1 - t0):.3f} ms, copy done {1e3 * (t2 - t0):.3f} ms",
              flush=True)
