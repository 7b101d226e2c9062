// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) throughput on sm_100a, against the DFMA
// peak: evidence for the DMMA accumulate-and-multiply variant decision.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == -1.0) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int iters = 20000;
  for (int warps : {4, 8, 16}) {
    dmma_loop<<<148, warps * 32>>>(o, iters);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dmma_loop<<<148, warps * 32>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 148.0 * warps * (double)iters * 4 * (8 * 8 * 4 * 2);
    printf("DMMA m8n8k4 warps/SM=%2d: %.2f TF/s (%s)\n", warps, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
