"""H2D bandwidth from pinned memory (T's 3.2 GB A): cudaHostAlloc'd (torch pin_memory) vs an
anonymous mapping advised for transparent huge pages and registered with cudaHostRegister;
each copied twice, with a 1 GB D2H in between (as the per-block Q_i / B_i copies do)."""
import ctypes
import mmap

import numpy as np
import torch

n = 20000 * 20000
nbytes = n * 8
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libcudart = ctypes.CDLL("libcudart.so.12") if False else None


def thp_pinned(nbytes):
    mm = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    buf = (ctypes.c_char * len(mm)).from_buffer(mm)
    addr = ctypes.addressof(buf)
    aligned = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
    MADV_HUGEPAGE = 14
    r = libc.madvise(ctypes.c_void_p(aligned), ctypes.c_size_t(nbytes), MADV_HUGEPAGE)
    arr = np.frombuffer(mm, dtype=np.uint8, count=nbytes, offset=aligned - addr)
    arr[::4096] = 0  # touch
    t = torch.from_numpy(arr.view(np.float64))
    err = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 0)
    return t, mm, buf, r, err


d = torch.empty(n, dtype=torch.float64, device="cuda")
junk_d = torch.empty(1 << 27, dtype=torch.float64, device="cuda")
junk_h = torch.empty(1 << 27, dtype=torch.float64).pin_memory()


def h2d(h, label):
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{label} rep {rep}: {ms:7.2f} ms  {nbytes / ms / 1e6:6.1f} GB/s", flush=True)
        junk_h.copy_(junk_d, non_blocking=True)  # 1 GB D2H in between
        torch.cuda.synchronize()


h = torch.empty(n, dtype=torch.float64).pin_memory()
h.fill_(1.0)
h2d(h, "cudaHostAlloc")
del h
t, mm, buf, r, err = thp_pinned(nbytes)
print("madvise", r, "cudaHostRegister", err, flush=True)
h2d(t, "THP+register ")
try:
    print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
except Exception as e:
    print("thp?", e)
