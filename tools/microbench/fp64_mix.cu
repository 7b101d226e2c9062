// FP64 pipe throughput by instruction mix (DFMA only, DMUL only, DADD only, rotation mix).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void mix(double* out, int iters, double a, double b) {
  double x[8], y[8], z[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { x[c] = threadIdx.x + c; y[c] = c * 0.5 + threadIdx.x * 1e-3; z[c] = 1e-3 * c; }
  const double cr = 0.999 + 1e-9 * threadIdx.x, sr = 0.001 + 1e-9 * threadIdx.x;  // per-thread registers
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (MODE == 0) { x[c] = fma(x[c], a, b); y[c] = fma(y[c], a, b); }          // 2 DFMA
      if (MODE == 1) { x[c] = x[c] * a; y[c] = y[c] * b; }                        // 2 DMUL
      if (MODE == 2) { x[c] = x[c] + a; y[c] = y[c] + b; }                        // 2 DADD
      if (MODE == 4) { x[c] = fma(x[c], y[c], z[c]); }                          // DFMA, 3 register operands
      if (MODE == 5) { x[c] = fma(x[c], y[(c + 1) & 7], x[(c + 3) & 7]); }       // DFMA, 3 registers, shared
      if (MODE == 6) {                                                            // rotation, c/s in registers
        double cx = __dmul_rn(cr, x[c]), sx = __dmul_rn(sr, x[c]);
        double nx = __fma_rn(sr, y[c], cx), ny = __fma_rn(cr, y[c], -sx);
        x[c] = nx; y[c] = ny;
      }
      if (MODE == 3) {                                                            // rotation: 2 DMUL + 2 DFMA
        double cx = __dmul_rn(a, x[c]), sx = __dmul_rn(b, x[c]);
        double nx = __fma_rn(b, y[c], cx), ny = __fma_rn(a, y[c], -sx);
        x[c] = nx; y[c] = ny;
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c] + y[c];
  if (s == 1.2345) out[0] = s;
}
template <int MODE>
void run(const char* name, int instr_per_iter_per_chain) {
  double* o; cudaMalloc(&o, 8);
  int blocks = 148 * 4, threads = 256, iters = 4000;
  mix<MODE><<<blocks, threads>>>(o, iters, 0.999, 0.001);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<MODE><<<blocks, threads>>>(o, iters, 0.999, 0.001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warp_instr = (double)blocks * threads / 32 * iters * 8 * instr_per_iter_per_chain;
  double per_smsp_cycle = warp_instr / (148.0 * 4) / (ms * 1e-3 * 1.965e9);
  printf("%-22s %.3f warp-FP64-instr per SMSP-cycle (at 1.965 GHz)\n", name, per_smsp_cycle);
}
int main() {
  run<0>("DFMA only", 2); run<1>("DMUL only", 2); run<2>("DADD only", 2); run<3>("rotation 2DMUL+2DFMA", 4);
  run<4>("DFMA 3 reg operands", 1); run<5>("DFMA 3 regs shared", 1); run<6>("rotation, c/s in regs", 4);
  return 0;
}
