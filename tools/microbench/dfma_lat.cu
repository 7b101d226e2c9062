// DFMA dependent-chain latency and ILP sweep on one SMSP (one warp per CTA, one CTA)
// and with 1..4 warps per SMSP: how many independent DFMA chains per warp saturate the
// FP64 pipe. Prints cycles per DFMA per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void chain(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == -1.0) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (double)(t1 - t0) / ((double)iters * ILP);
}
template <int ILP>
void run(int warps_per_smsp) {
  double* o; cudaMalloc(&o, 16);
  int iters = 20000;
  chain<ILP><<<148, 128 * warps_per_smsp>>>(o, iters, 0.999, 1e-3);
  chain<ILP><<<148, 128 * warps_per_smsp>>>(o, iters, 0.999, 1e-3);
  cudaDeviceSynchronize();
  double h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("ILP=%2d warps/SMSP=%d: %.2f cycles per DFMA per warp (pipe-bound floor = 2*warps = %d)\n", ILP,
         warps_per_smsp, h[1], 2 * warps_per_smsp);
  cudaFree(o);
}
int main() {
  for (int w = 1; w <= 4; ++w) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); run<16>(w); }
  return 0;
}
