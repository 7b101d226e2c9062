// Steady-state ceiling of the scaled-form block body as a function of rows per thread
// (R), lanes per unit (KB) and warps per SM, with the register budget that warp count
// allows (launch bounds). Coefficients: LDS.128 broadcast from a rotating smem buffer;
// ring I/O: one column in (LDS) and one out (STS) per wave; one scale DMUL per row per wave.
#include <cstdio>
#include <cuda_runtime.h>
template <int K, int KB, int R, int NT, int V, int PAIR>
__global__ void __launch_bounds__(NT, 1) body(double* out, int nblocks, int cw) {
  extern __shared__ double2 sm[];
  double2* coef = sm;
  double* io = (double*)(sm + cw * K);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < cw * K; i += blockDim.x) {
    double th = 0.001 * i; coef[i] = make_double2(0.1 * sin(th), -0.1 * cos(th));
  }
  double* myio = io + warp * 32 * R * (K + 1);
  const double* inio = io + (warp ^ 1) * 32 * R * (K + 1);  // another warp's slot: no store-to-load forwarding
  for (int i = lane; i < 32 * R * (K + 1); i += 32) myio[i] = 1.0 + i;
  __syncthreads();
  double w[R][K + 1];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int s = 0; s <= K; ++s) w[r][s] = 0.5 * s + r;
  int cbase = 0;
  for (int b = 0; b < nblocks; ++b) {
    const double2* cb = coef + cbase;
#pragma unroll
    for (int u = 0; u <= K; ++u) {
      double nv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) nv[r] = *(volatile const double*)&inio[(((u + 3) % (K + 1)) * R + r) * 32 + lane];
      const double sc = cb[(K + 1) * KB + u / 2].x;
#pragma unroll
      for (int r = 0; r < R; ++r) myio[(u * R + r) * 32 + lane] = w[r][u] * sc;
#pragma unroll
      for (int r = 0; r < R; ++r) w[r][u] = nv[r];
#pragma unroll
      for (int l = 0; l < KB; ++l) {
        const double2 cs = V == 0 ? cb[u * KB + l] : (V == 1 ? cb[u * KB] : make_double2(0.01 * (l + 1), -0.02 * (u + 1)));
        const int sx = ((u - 1 - l) % (K + 1) + 2 * (K + 1)) % (K + 1);
        const int sy = (sx + 1) % (K + 1);
if (PAIR) {
          double xo[R];
#pragma unroll
          for (int r = 0; r < R; ++r) xo[r] = w[r][sx];
#pragma unroll
          for (int r = 0; r < R; ++r) w[r][sx] = fma(cs.x, w[r][sy], xo[r]);
#pragma unroll
          for (int r = 0; r < R; ++r) w[r][sy] = fma(cs.y, xo[r], w[r][sy]);
        } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double x = w[r][sx], y = w[r][sy];
          w[r][sx] = fma(cs.x, y, x);
          w[r][sy] = fma(cs.y, x, y);
        }
        }
      }
    }
    cbase += (K + 1) * KB + 8;
    if (cbase + 2 * ((K + 1) * KB + 8) > cw * K) cbase = 0;
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int q = 0; q <= K; ++q) s += w[r][q];
  if (s == 1.2345) out[0] = s;
}
template <int K, int KB, int R, int NT, int V = 0, int PAIR = 0>
void run() {
  const int warps = NT / 32;
  int cw = 64 * (K + 1);
  size_t smem = cw * K * 16 + (size_t)warps * 32 * R * (K + 1) * 8;
  auto kern = body<K, KB, R, NT, V, PAIR>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
  double* o; cudaMalloc(&o, 8);
  int grid = 148, nb = 3000;
  kern<<<grid, NT, smem>>>(o, nb, cw);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<grid, NT, smem>>>(o, nb, cw);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double elems = (double)grid * NT * R * (double)nb * (K + 1) * KB;
  double fl = 6.0 * elems;
  double fp64 = elems / 32.0 * 2.0 + (double)grid * warps * R * nb * (K + 1);
  double util = fp64 / (148.0 * 4 * 0.5 * (ms * 1e-3 * 1.965e9));
  printf("P%d V%d KB=%d R=%d warps/SM=%2d regs=%3d spill=%zu: %6.2f counted TF/s (%5.1f%% of 34.2) FP64 pipe %.1f%% %s\n", PAIR, V, KB, R,
         warps, fa.numRegs, (size_t)fa.localSizeBytes, fl / ms / 1e9, fl / ms / 1e9 / 34.2 * 100, util * 100,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}
int main() {
  run<8, 8, 2, 384, 0, 0>(); run<8, 8, 2, 384, 0, 1>();
  run<8, 8, 3, 384, 0, 0>(); run<8, 8, 3, 384, 0, 1>();
  run<8, 8, 4, 256, 0, 0>(); run<8, 8, 4, 256, 0, 1>();
  run<8, 7, 2, 384, 0, 1>(); run<8, 6, 2, 384, 0, 1>();
  return 0;
}
