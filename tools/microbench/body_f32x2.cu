// fp32 block body: scalar FFMA with two rows per thread (records of two lanes per 16 bytes,
// the layout the fp32 pipeline uses) against packed fma.rn.f32x2 (sm_100 FFMA2) with the
// thread's two rows in one 64-bit register and duplicated (tau, tau) records.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) { u64 d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
template <int K, int NT, int V>
__global__ void __launch_bounds__(NT, 1) body(float* out, int nblocks, int cw) {
  extern __shared__ float4 sm[];
  float4* coef = sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < cw * K; i += blockDim.x) { float th = 0.001f * i; coef[i] = make_float4(0.1f * sinf(th), 0.1f * sinf(th), -0.1f * cosf(th), -0.1f * cosf(th)); }
  float* io = (float*)(sm + cw * K);
  float* myio = io + warp * 64 * (K + 1);
  const float* inio = io + (warp ^ 1) * 64 * (K + 1);
  for (int i = lane; i < 64 * (K + 1); i += 32) myio[i] = 1.0f + i;
  __syncthreads();
  int cbase = 0;
  if (V == 0) {
    float w[2][K + 1];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int s = 0; s <= K; ++s) w[r][s] = 0.5f * s + r;
    for (int b = 0; b < nblocks; ++b) {
      const float4* cb = coef + cbase;
#pragma unroll
      for (int u = 0; u <= K; ++u) {
        float nv[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) nv[r] = *(volatile const float*)&inio[(((u + 3) % (K + 1)) * 2 + r) * 32 + lane];
        const float sc = cb[(K + 1) * K / 2 + u / 4].x;
#pragma unroll
        for (int r = 0; r < 2; ++r) myio[(u * 2 + r) * 32 + lane] = w[r][u] * sc;
#pragma unroll
        for (int r = 0; r < 2; ++r) w[r][u] = nv[r];
#pragma unroll
        for (int l = 0; l < K; ++l) {
          const float4 c4 = cb[u * (K / 2) + l / 2];
          const float t1 = (l & 1) ? c4.z : c4.x, t2 = (l & 1) ? c4.w : c4.y;
          const int sx = ((u - 1 - l) % (K + 1) + 2 * (K + 1)) % (K + 1), sy = (sx + 1) % (K + 1);
#pragma unroll
          for (int r = 0; r < 2; ++r) { const float x = w[r][sx], y = w[r][sy]; w[r][sx] = fmaf(t1, y, x); w[r][sy] = fmaf(t2, x, y); }
        }
      }
      cbase += (K + 1) * K / 2 + 8;
      if (cbase + 2 * ((K + 1) * K + 8) > cw * K) cbase = 0;
    }
    float s = 0;
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int q = 0; q <= K; ++q) s += w[r][q];
    if (s == 1.2345f) out[0] = s;
  } else {
    u64 w[K + 1];
#pragma unroll
    for (int s = 0; s <= K; ++s) w[s] = 0x3f0000003f800000ull + s * 0x0000100000001000ull;
    u64* myio2 = (u64*)myio;
    const u64* inio2 = (const u64*)inio;
    for (int b = 0; b < nblocks; ++b) {
      const float4* cb = coef + cbase;
#pragma unroll
      for (int u = 0; u <= K; ++u) {
        const u64 nv = *(volatile const u64*)&inio2[((u + 3) % (K + 1)) * 32 + lane];
        const u64 sc = *(const u64*)&cb[(K + 1) * K + u / 2];
        myio2[u * 32 + lane] = fmul2(w[u], sc);
        w[u] = nv;
#pragma unroll
        for (int l = 0; l < K; ++l) {
          const ulonglong2 c2 = *(const ulonglong2*)&cb[u * K + l];
          const int sx = ((u - 1 - l) % (K + 1) + 2 * (K + 1)) % (K + 1), sy = (sx + 1) % (K + 1);
          const u64 x = w[sx], y = w[sy];
          w[sx] = ffma2(c2.x, y, x);
          w[sy] = ffma2(c2.y, x, y);
        }
      }
      cbase += (K + 1) * K + 8;
      if (cbase + 2 * ((K + 1) * K + 8) > cw * K) cbase = 0;
    }
    u64 s = 0;
#pragma unroll
    for (int q = 0; q <= K; ++q) s ^= w[q];
    if (s == 12345ull) out[0] = 1.0f;
  }
}
template <int K, int NT, int V>
void run() {
  const int warps = NT / 32;
  int cw = 64 * (K + 1);
  size_t smem = cw * K * 16 + (size_t)warps * 64 * (K + 1) * 4;
  auto kern = body<K, NT, V>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
  float* o; cudaMalloc(&o, 8);
  int grid = 148, nb = 3000;
  kern<<<grid, NT, smem>>>(o, nb, cw);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<grid, NT, smem>>>(o, nb, cw);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double elems = (double)grid * NT * 2 * (double)nb * (K + 1) * K;
  double fl = 6.0 * elems;
  printf("%s K=%d warps/SM=%2d regs=%3d: %6.2f counted TF/s (%5.1f%% of the 72.3 TF/s FFMA peak) %s\n", V ? "f32x2 " : "scalar", K,
         warps, fa.numRegs, fl / ms / 1e9, fl / ms / 1e9 / 72.3 * 100, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}
int main() {
  run<8, 512, 0>(); run<8, 512, 1>(); run<8, 384, 0>(); run<8, 384, 1>();
  return 0;
}
