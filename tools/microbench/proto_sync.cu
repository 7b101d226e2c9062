// Cost of the per-block hand-off protocol on the steady-state block (K=8, R=2, fast):
// P0 no sync; P1 + coefficient bulk copy + mbarrier wait per block; P2 + warp barrier and
// lane-0 release/arrive per block; P3 + an (already complete) mbarrier wait on the ring.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void marrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(dst)), "l"(src), "r"(bytes), "r"(su(bar)) : "memory");
}
template <int K, int R, int MODE>
__global__ void __launch_bounds__(512, 1) steady(double* out, const double2* __restrict__ gcoef, int nblocks, int ncb, int kb = K) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
  double2* cbuf = reinterpret_cast<double2*>(smraw) + warp * 2 * (K + 1) * K;
  double* io = reinterpret_cast<double*>(reinterpret_cast<double2*>(smraw) + NW * 2 * (K + 1) * K) + warp * 3 * 32 * R * (K + 1);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(reinterpret_cast<double2*>(smraw) + NW * 2 * (K + 1) * K) + NW * 3 * 32 * R * (K + 1)) + warp * 8;
  uint32_t* counter = reinterpret_cast<uint32_t*>(bars + 6);
  if (lane == 0) { for (int i = 0; i < 5; ++i) minit(bars + i, 1); *counter = 0; }
  for (int i = lane; i < 2 * (K + 1) * K; i += 32) cbuf[i] = gcoef[i];
  for (int i = lane; i < 3 * 32 * R * (K + 1); i += 32) io[i] = 1.0 + 1e-3 * i;
  __syncwarp();
  double w[R][K + 1];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int s = 0; s <= K; ++s) w[r][s] = 0.5 * s + r;
  uint32_t cseq = 0;
  if (MODE >= 1 && lane == 0) bulk(cbuf, gcoef, (K + 1) * K * 16, &bars[3]);
  for (int b = 0; b < nblocks; ++b) {
    if (MODE >= 1) {
      if (lane == 0) bulk(cbuf + ((cseq + 1) & 1) * (K + 1) * K, gcoef + (size_t)((b + 1) % ncb) * (K + 1) * K, (K + 1) * K * 16, &bars[3 + ((cseq + 1) & 1)]);
      mwait(&bars[3 + (cseq & 1)], (cseq >> 1) & 1);
    }
    if (MODE == 3) mwait(&bars[b % 3], ((b / 3) & 1));
    const double2* cb = cbuf + (MODE >= 1 ? (cseq & 1) : 0) * (K + 1) * K;
    double* islot = io + (b % 3) * 32 * R * (K + 1);
#pragma unroll
    for (int u = 0; u <= K; ++u) {
#pragma unroll
      for (int r = 0; r < R; ++r) islot[u * 32 * R + lane + 32 * r] = w[r][u];
#pragma unroll
      for (int r = 0; r < R; ++r) w[r][u] = islot[u * 32 * R + lane + 32 * r + 1];
#pragma unroll
      for (int l = 0; l < K; ++l) {
        if (MODE == 5 && l >= kb) continue;
        const double2 cs = cb[u * K + l];
        const int sx = ((u - l - 1) % (K + 1) + (K + 1)) % (K + 1), sy = (sx + 1) % (K + 1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double x = w[r][sx], y = w[r][sy];
          const double cx = __dmul_rn(cs.x, x), sxx = __dmul_rn(cs.y, x);
          w[r][sx] = __fma_rn(cs.y, y, cx);
          w[r][sy] = __fma_rn(cs.x, y, -sxx);
        }
      }
    }
    if (MODE >= 2) {
      __syncwarp();
      if (lane == 0) {
        asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(su(counter)), "r"(b + 1) : "memory");
        marrive(&bars[(b + 1) % 3]);
      }
    }
    ++cseq;
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int q = 0; q <= K; ++q) s += w[r][q];
  if (s == 1.2345) out[0] = s;
}
template <int MODE, int R = 2, int K = 8>
void run(int warps, int kb = K) {
  size_t smem = (size_t)warps * (2 * (K + 1) * K * 16 + 3 * 32 * R * (K + 1) * 8 + 64);
  cudaFuncSetAttribute(steady<K, R, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int ncb = 64;
  double2* gc; cudaMalloc(&gc, (size_t)ncb * (K + 1) * K * 16);
  cudaMemset(gc, 0, (size_t)ncb * (K + 1) * K * 16);
  double* o; cudaMalloc(&o, 8);
  int nb = 2000;
  steady<K, R, MODE><<<148, warps * 32, smem>>>(o, gc, 10, ncb);
  if (MODE >= 3) {}  // the ring barrier of block b is arrived at the end of block b-1 (self-produced)
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  steady<K, R, MODE><<<148, warps * 32, smem>>>(o, gc, nb, ncb, kb);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 6.0 * 148 * warps * 32 * R * (double)nb * (K + 1) * kb;
  printf("kb %d K %d R %d MODE %d warps/SM %2d: %.2f TF/s (%.1f%% of 34.15)  %s\n", kb, K, R, MODE, warps, fl / ms / 1e9, fl / ms / 1e9 / 34.15 * 100,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int w : {8, 12}) { run<2>(w); run<5>(w, 8); run<5>(w, 7); run<5>(w, 6); run<2, 2, 7>(w); run<2, 2, 6>(w); }
  return 0;
}
