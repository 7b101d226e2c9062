// Steady-state ceiling of the unrolled block body, standard fast form vs the scaled
// (fast Givens) form: register window of K+1 columns x R rows per thread, KB lanes,
// coefficients from smem (LDS.128 broadcast), one column in / one out per wave through
// smem. No HBM traffic, no inter-warp protocol. Reports counted TF/s (6 flops per
// rotation element) and FP64 pipe utilisation (DFMA/DMUL issue vs 0.5/cycle/SMSP).
#include <cstdio>
#include <cuda_runtime.h>
template <int K, int KB, int R, bool SCALED, int VAR = 0>
__global__ void __launch_bounds__(512, 1) steady(double* out, int nblocks, int cw) {
  extern __shared__ double2 sm[];
  double2* coef = sm;
  double* io = (double*)(sm + cw * K);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < cw * K; i += blockDim.x) {
    double th = 0.001 * i; coef[i] = make_double2(cos(th) * 0.9, sin(th) * 0.1);
  }
  double* myio = io + warp * 32 * R * (K + 1);
  for (int i = lane; i < 32 * R * (K + 1); i += 32) myio[i] = 1.0 + i;
  __syncthreads();
  double w[R][K + 1];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int s = 0; s <= K; ++s) w[r][s] = 0.5 * s + r;
  int cbase = 0;
  double2 cn[KB];  // VAR 3: next wave's coefficients, loaded one wave ahead
#pragma unroll
  for (int l = 0; l < KB; ++l) cn[l] = coef[l];
  for (int b = 0; b < nblocks; ++b) {
#pragma unroll
    for (int u = 0; u <= K; ++u) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double v = SCALED ? w[r][u] * coef[cbase + u].x : w[r][u];
        if (VAR != 1) myio[(u * R + r) * 32 + lane] = v;
        else w[r][u] = v;
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (VAR != 1) w[r][u] = myio[(((u + 3) % (K + 1)) * R + r) * 32 + lane];
      double2 cc[KB];
#pragma unroll
      for (int l = 0; l < KB; ++l) cc[l] = cn[l];
      if (VAR == 3) {
        const int nb = (u == K) ? ((cbase + (K + 1) * KB + 16 > cw * K - (K + 1) * KB) ? 0 : cbase + (K + 1) * KB) : cbase;
        const int nu = (u == K) ? 0 : u + 1;
#pragma unroll
        for (int l = 0; l < KB; ++l) cn[l] = coef[nb + nu * KB + l];
      }
#pragma unroll
      for (int l = 0; l < KB; ++l) {
        const double2 cs = VAR == 2 ? make_double2(0.999 - 1e-4 * l, 1e-4 * u) : (VAR == 3 ? cc[l] : coef[cbase + u * KB + l]);
        const int sx = ((u - 1 - l) % (K + 1) + 2 * (K + 1)) % (K + 1);
        const int sy = (sx + 1) % (K + 1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double x = w[r][sx], y = w[r][sy];
          if (SCALED) {
            w[r][sx] = fma(cs.x, y, x);
            w[r][sy] = fma(cs.y, x, y);
          } else {
            const double cx = cs.x * x, sxx = cs.y * x;
            w[r][sx] = fma(cs.y, y, cx);
            w[r][sy] = fma(cs.x, y, -sxx);
          }
        }
      }
    }
    cbase += (K + 1) * KB;
    if (cbase + (K + 1) * KB + 16 > cw * K) cbase = 0;
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int q = 0; q <= K; ++q) s += w[r][q];
  if (s == 1.2345) out[0] = s;
}
template <int K, int KB, int R, bool SCALED, int VAR = 0>
void run(int warps) {
  int cw = 64 * (K + 1);
  size_t smem = cw * K * 16 + (size_t)warps * 32 * R * (K + 1) * 8;
  cudaFuncSetAttribute(steady<K, KB, R, SCALED, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double* o; cudaMalloc(&o, 8);
  int grid = 148, nb = 4000;
  steady<K, KB, R, SCALED, VAR><<<grid, warps * 32, smem>>>(o, nb, cw);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  steady<K, KB, R, SCALED, VAR><<<grid, warps * 32, smem>>>(o, nb, cw);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double elems = (double)grid * warps * 32 * R * (double)nb * (K + 1) * KB;  // rotation elements
  double fl = 6.0 * elems;
  double fp64_instr = elems / 32.0 * (SCALED ? 2.0 : 4.0) + (SCALED ? (double)grid * warps * R * nb * (K + 1) : 0);
  double cycles = ms * 1e-3 * 1.965e9;
  double util = fp64_instr / (148.0 * 4 * 0.5 * cycles);
  printf("KB=%d R=%d var%d %s warps/SM=%2d: %6.2f counted TF/s (%5.1f%% of 34.2)  FP64 pipe %.1f%%  %s\n", KB, R,
         VAR, SCALED ? "scaled  " : "standard", warps, fl / ms / 1e9, fl / ms / 1e9 / 34.2 * 100, util * 100,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}
int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == '3') { run<8, 7, 3, true, 0>(12); return 0; }
  if (argc > 1 && argv[1][0] == '2') { run<8, 7, 2, true, 0>(12); return 0; }
  run<8, 8, 2, true, 0>(8); run<8, 8, 2, true, 0>(12); run<8, 8, 2, true, 0>(16);
  run<8, 8, 2, true, 1>(12); run<8, 8, 2, true, 2>(12); run<8, 8, 2, true, 3>(12);
  run<8, 8, 3, true, 0>(8); run<8, 8, 3, true, 0>(12);
  run<8, 8, 4, true, 0>(8);
  run<8, 8, 2, false, 0>(12);
  return 0;
}
