// DFMA issue rate vs operand sources: how many distinct vector-register operands a DFMA
// can read per issue without slowing the FP64 pipe (register-file read bandwidth).
#include <cstdio>
#include <cuda_runtime.h>
template <int P>
__global__ void __launch_bounds__(256, 1) k(double* out, int iters, double p0, double p1) {
  double x[8], y[8], c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; y[i] = 0.5 * i + threadIdx.x; c[i] = 1e-3 * (i + threadIdx.x); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (P == 0) x[i] = fma(c[i], y[i], x[i]);            // 3 distinct registers
      if (P == 1) x[i] = fma(c[0], y[i], x[i]);            // shared multiplier register (reuse)
      if (P == 2) x[i] = fma(p0, y[i], x[i]);              // multiplier from constant bank
      if (P == 3) { const double xo = x[i]; x[i] = fma(c[i], y[i], x[i]); y[i] = fma(c[(i + 1) & 7], xo, y[i]); }
      if (P == 4) x[i] = fma(x[i], y[i], p1);              // 2 registers + constant addend
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + y[i];
  if (s == -1.0) out[0] = s;
}
template <int P>
void run() {
  double* o; cudaMalloc(&o, 8);
  int iters = 20000;
  k<P><<<148, 256>>>(o, iters, 1e-3, 0.5);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<P><<<148, 256>>>(o, iters, 1e-3, 0.5);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double dfma = 148.0 * 8 * (double)iters * 8 * (P == 3 ? 2 : 1);
  double util = dfma / (148.0 * 4 * 0.5 * ms * 1e-3 * 1.965e9);
  printf("P%d: FP64 pipe %.1f%%\n", P, 100 * util);
}
int main() { run<0>(); run<1>(); run<2>(); run<3>(); run<4>(); return 0; }
