"""cuBLAS FP64 yardsticks via torch (library GEMM, measurement only; never on the product path).

Prints JSON: DGEMM TFLOP/s at 8192^3 and at the randQB block shapes of the target
config T (20000 x 20000, b = 256): A @ Omega, Q^T @ A, A - Q @ B.
"""
import json
import torch


def bench(fn, flops, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return flops / best * 1e-12


def main():
    dev = torch.device("cuda:0")
    res = {"gpu": torch.cuda.get_device_name(0)}
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    res["dgemm_8192_tflops"] = bench(lambda: a @ b, 2.0 * n ** 3)
    del a, b
    m = nn = 20000
    w = 256
    A = torch.randn(nn, m, dtype=torch.float64, device=dev).t()  # column-major m x n
    Om = torch.randn(nn, w, dtype=torch.float64, device=dev)
    Q = torch.randn(w, m, dtype=torch.float64, device=dev).t()
    B = torch.randn(w, nn, dtype=torch.float64, device=dev)
    res["dgemm_A_Omega_tflops"] = bench(lambda: A @ Om, 2.0 * m * nn * w)
    res["dgemm_QtA_tflops"] = bench(lambda: Q.t() @ A, 2.0 * m * nn * w)
    res["dgemm_downdate_tflops"] = bench(lambda: torch.addmm(A, Q, B, alpha=-1.0), 2.0 * m * nn * w)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
