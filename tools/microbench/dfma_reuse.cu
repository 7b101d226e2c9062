// How much of the 3-register-operand DFMA penalty (RF read bandwidth: 3 cycles per RRR DFMA
// against the pipe's 2) the operand reuse cache recovers when G consecutive DFMAs of a warp
// share their multiplier register, at 1..4 warps per SM sub-partition.
#include <cstdio>
#include <cuda_runtime.h>
template <int G, int NT>
__global__ void __launch_bounds__(NT, 1) k(double* out, int iters) {
  double x[16], y[16], c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { x[i] = threadIdx.x + i; y[i] = 0.5 * i + threadIdx.x; c[i] = 1e-3 * (i + threadIdx.x); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(c[(i / G) * G], y[i], x[i]);
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = fma(c[(i / G) * G + (G > 1 ? 1 : 0)], x[i], y[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i] + y[i];
  if (s == -1.0) out[0] = s;
}
template <int G, int NT>
void run() {
  double* o; cudaMalloc(&o, 8);
  int iters = 20000;
  k<G, NT><<<148, NT>>>(o, iters);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<G, NT><<<148, NT>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double dfma = 148.0 * (NT / 32) * (double)iters * 32;
  double util = dfma / (148.0 * 4 * 0.5 * ms * 1e-3 * 1.965e9);
  printf("group=%d warps/SMSP=%d: FP64 pipe %.1f%%\n", G, NT / 128, 100 * util);
  cudaFree(o);
}
int main() {
  run<1, 128>(); run<2, 128>(); run<4, 128>(); run<8, 128>();
  run<1, 256>(); run<2, 256>(); run<4, 256>(); run<8, 256>();
  run<1, 384>(); run<2, 384>(); run<4, 384>(); run<8, 384>();
  run<1, 512>(); run<2, 512>(); run<4, 512>(); run<8, 512>();
  return 0;
}
