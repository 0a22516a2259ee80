// FP64 throughput microbenchmarks for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA.
// Used once to fix the FP64 roofline denominator; not product code.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dmma_m16n8k8(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = a0, a2 = a0, a3 = a0, b0 = 1.0, b1 = 1.0;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dfma_chain(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
static double timeit(K kern, int grid, int block, double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<grid, block>>>(out, iters / 10);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  kern<<<grid, block>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e-3;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    int block = 32 * wpb, grid = sms * 2;
    double t = timeit(dmma_m8n8k4<8>, grid, block, out, iters);
    double flops = 2.0 * 256 * 8 * (double)iters * grid * wpb;
    printf(", \"dmma_m8n8k4_w%d_tflops\": %.3f", wpb, flops / t * 1e-12);
    t = timeit(dmma_m16n8k8<4>, grid, block, out, iters);
    flops = 2.0 * 1024 * 4 * (double)iters * grid * wpb;
    printf(", \"dmma_m16n8k8_w%d_tflops\": %.3f", wpb, flops / t * 1e-12);
    t = timeit(dfma_chain<8>, grid, block, out, iters);
    flops = 2.0 * 32 * 8 * (double)iters * grid * wpb;
    printf(", \"dfma_w%d_tflops\": %.3f", wpb, flops / t * 1e-12);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
