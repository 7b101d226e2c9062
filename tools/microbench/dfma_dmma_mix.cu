// Do the FP64 FMA pipe (DFMA) and the FP64 tensor cores (DMMA) run concurrently on B200?
// Warps [0, nd) of each CTA run independent DFMA chains, warps [nd, nw) DMMA chains; the
// two throughputs are reported separately and together. If they add, a kernel could split
// its rotations between the register-window path and the window-product path.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mix(double* out, int iters, int nd) {
  const int warp = threadIdx.x >> 5;
  if (warp < nd) {
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], 0.999, 0.001);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c];
    if (s == -1.0) out[0] = s;
  } else {
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
    double c[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = threadIdx.x;
    for (int it = 0; it < iters / 4; ++it) {
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
}

int main() {
  double* o;
  cudaMalloc(&o, 8);
  const int iters = 40000;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Cfg { int nd, nm; } cfgs[] = {{8, 0}, {0, 8}, {8, 8}, {4, 4}, {12, 4}, {4, 12}};
  for (auto cfg : cfgs) {
    const int nw = cfg.nd + cfg.nm;
    mix<<<sms, nw * 32>>>(o, iters, cfg.nd);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mix<<<sms, nw * 32>>>(o, iters, cfg.nd);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dfma = (double)sms * cfg.nd * 32 * (double)iters * 8 * 2;
    const double dmma = (double)sms * cfg.nm * (double)(iters / 4) * 4 * 512;
    printf("DFMA warps %2d + DMMA warps %2d: %.2f ms  DFMA %.2f TF/s + DMMA %.2f TF/s = %.2f TF/s (%s)\n", cfg.nd,
           cfg.nm, ms, dfma / ms / 1e9, dmma / ms / 1e9, (dfma + dmma) / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
