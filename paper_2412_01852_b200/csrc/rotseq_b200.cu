// rotseq_b200.cu — B200-native (sm_100a) application of a rotation sequence to a
// column-major matrix. C-ABI declared in include/rotseq_b200.h.
//
// What the reference does (Python + numba, CPU):
//   semantic definition  _naive_py            /root/reference/pkg/src/rotseq/core.py:195-205
//   2x2 formulas         _rot_cols/_refl_cols  core.py:130-149
//   wavefront schedule   _span_impl            core.py:152-172 (wave t, lane l -> (t-l, p0+l))
//   hot loop             _kernel_chunk_py      blocking.py:342-397 (startup triangle,
//                        n_b-wave windows with wave-major coefficient tiles, shutdown triangle)
//   threads over rows    _run_row_ranges       blocking.py:518-526
//
// The B200 design:
//   * A "unit" is (tile of 32*R owners, band of K consecutive sweeps). One warp runs one
//     unit: every lane owns R rows (right side; columns for the left side) and keeps a
//     (K+1)-column window of them in registers. Waves are processed in blocks of K+1 so
//     the window rotates through fixed registers (slot = column mod (K+1)) — true register
//     residency, which the reference only models (SURVEY §2 note, kernels.py:135-147).
//   * Bands of one tile are chained warp-to-warp through shared-memory rings guarded by
//     mbarriers: warp w streams finished columns of band b to warp w+1 (band b+1), so A
//     crosses HBM once per chain instead of once per band.
//   * Coefficients are repacked once per call into a band-major, wave-major stream of
//     (c,s) pairs (the GPU analogue of the reference's per-window coefficient gather,
//     blocking.py:364-373) and staged per block by cp.async.bulk (TMA bulk copy) into a
//     per-warp double buffer; every lane reads them as broadcast LDS.128.
//   * A persistent grid of one CTA per SM splits the unit list (tile-major) evenly; a
//     chain that crosses a CTA boundary (or a round boundary inside a CTA) is handed off
//     through A itself (in place) with per-unit release/acquire progress flags in global
//     memory. All CTAs are co-resident (cooperative launch), so waits always make progress.
//   * strict mode uses __dmul_rn/__dadd_rn/__dsub_rn in the reference's exact expression
//     shape (no contraction => bit-identical to the reference strict build); fast mode uses
//     2 DMUL + 2 DFMA per rotation element (the 4-instruction minimum for 6 flops).

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include "rotseq_b200.h"

#define RS_VERSION 10000

namespace {

// ------------------------------------------------------------------------------------
// compile-time geometry
// ------------------------------------------------------------------------------------
constexpr int kK = 8;          // sweeps per band (lanes of the wavefront)
constexpr int kR = 2;          // owners (rows) per thread
#ifndef RS_STAGES
#define RS_STAGES 3
#endif
constexpr int kStages = RS_STAGES;  // ring depth in chunks of K+1 columns
constexpr int kMaxWarps = 16;  // warps per CTA upper bound (launch bounds)
constexpr int kTileOwners = 32 * kR;
constexpr int kCtlWords = kStages + 3;  // per-warp control words (see rs_pipeline_kernel)
constexpr int kFlagEvery = 8;   // hand-off progress is published every 8 blocks (fence cost)
constexpr size_t kTrashBytes = 32 * kR * 8;  // scratch slot per lane for rows past the matrix

enum : int { SRC_RING = 0, SRC_GLOBAL = 1, SRC_FLAG = 2 };
enum : int { DST_RING = 0, DST_GLOBAL = 1, DST_FLAG = 2 };

std::atomic<long long> g_launches{0};
thread_local std::string g_err;

rs_status fail(rs_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

// ------------------------------------------------------------------------------------
// coefficient records and arithmetic
// ------------------------------------------------------------------------------------
template <typename T, bool REFL>
struct Coef;
template <typename T>
struct alignas(2 * sizeof(T)) Coef<T, false> {
  T c, s;
};
template <typename T>
struct alignas(4 * sizeof(T)) Coef<T, true> {
  T s, d, e, pad;  // d = c - s, e = c + s (hoisted exactly as core.py:142-143)
};

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// Rotation (core.py:130-137):   x' = c*x + s*y ; y' = c*y - s*x
// Reflector (core.py:140-149):  w = s*(x+y) ; x' = w + d*x ; y' = w - e*y
template <typename T, bool STRICT>
__device__ __forceinline__ void rot2(T& x, T& y, T c, T s) {
  if constexpr (STRICT) {
    const T nx = add_rn(mul_rn(c, x), mul_rn(s, y));
    const T ny = sub_rn(mul_rn(c, y), mul_rn(s, x));
    x = nx;
    y = ny;
  } else {
    const T cx = mul_rn(c, x);
    const T sx = mul_rn(s, x);
    x = fma_rn(s, y, cx);
    y = fma_rn(c, y, -sx);
  }
}
template <typename T, bool STRICT>
__device__ __forceinline__ void refl2(T& x, T& y, T s, T d, T e) {
  const T w = mul_rn(s, add_rn(x, y));
  if constexpr (STRICT) {
    x = add_rn(w, mul_rn(d, x));
    y = sub_rn(w, mul_rn(e, y));
  } else {
    x = fma_rn(d, x, w);
    y = fma_rn(-e, y, w);
  }
}
template <typename T, bool STRICT, bool REFL>
__device__ __forceinline__ void xform(T& x, T& y, const Coef<T, REFL>& cf) {
  if constexpr (REFL) {
    refl2<T, STRICT>(x, y, cf.s, cf.d, cf.e);
  } else {
    rot2<T, STRICT>(x, y, cf.c, cf.s);
  }
}

// ------------------------------------------------------------------------------------
// PTX helpers: mbarrier, bulk copy, flags
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "RS_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra RS_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// One elected lane: expect `bytes` on `bar` and start a TMA bulk copy global -> shared.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// cp.async (LDGSTS) of one element; src_size 0 zero-fills (out-of-range rows/columns).
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src, bool valid) {
  if constexpr (sizeof(T) == 8) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 8 : 0)
                 : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 4 : 0)
                 : "memory");
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_shared(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_shared(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void wait_count(const uint32_t* p, uint32_t target) {
  while (ld_acquire_shared(p) < target) __nanosleep(32);
}
__device__ __forceinline__ uint32_t wait_flag(const uint32_t* p, uint32_t target) {
  uint32_t v;
  while ((v = ld_acquire(p)) < target) __nanosleep(64);
  return v;
}

// Debug-only instrumentation (compiled in with -DRS_TRACE; see rs_debug_set_trace).
// Each unit a warp runs writes one record of kTraceWords uint64 to
// g_trace[((cta * kMaxWarps + warp) * kTraceRounds + round) * kTraceWords]:
//   0 unit | src<<32 | dst<<40 | smid<<48, 1 globaltimer at unit start, 2 at unit end,
//   3 cycles waiting for self-fill / progress flags, 4 coefficient waits, 5 ring-full waits,
//   6 ring-space waits, 7 compute (run_block), 8 post-block hand-off work, 9 blocks.
constexpr int kTraceWords = 10;
constexpr int kTraceRounds = 32;
__device__ unsigned long long* g_trace = nullptr;
#ifdef RS_TRACE
__device__ __forceinline__ unsigned long long trace_clock() { return clock64(); }
__device__ __forceinline__ unsigned long long trace_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned trace_smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
#else
__device__ __forceinline__ unsigned long long trace_clock() { return 0; }
__device__ __forceinline__ unsigned long long trace_gtime() { return 0; }
__device__ __forceinline__ unsigned trace_smid() { return 0; }
#endif
struct TraceAcc {
  unsigned long long t0 = 0, c[6] = {0, 0, 0, 0, 0, 0};
};
__device__ __forceinline__ void trace_unit(int warp, int jr, long long u, int src, int dst, const TraceAcc& acc,
                                           int blocks) {
#ifdef RS_TRACE
  unsigned long long* t = g_trace;
  if (t != nullptr && (threadIdx.x & 31) == 0 && jr < kTraceRounds) {
    unsigned long long* rec = t + (((size_t)blockIdx.x * kMaxWarps + warp) * kTraceRounds + jr) * kTraceWords;
    rec[0] = (unsigned long long)u | ((unsigned long long)src << 32) | ((unsigned long long)dst << 40) |
             ((unsigned long long)trace_smid() << 48);
    rec[1] = acc.t0;
    rec[2] = trace_gtime();
    for (int i = 0; i < 6; ++i) rec[3 + i] = acc.c[i];
    rec[9] = (unsigned long long)blocks;
  }
#else
  (void)warp, (void)jr, (void)u, (void)src, (void)dst, (void)acc, (void)blocks;
#endif
}

// ------------------------------------------------------------------------------------
// kernel parameters
// ------------------------------------------------------------------------------------
struct PipeParams {
  void* A;               // element (owner o, wave-column v) at A + o*os + v*cs
  long long os;          // owner stride (elements)
  long long cs;          // wave-column stride (elements, negative for reverse order)
  long long owners;      // independent lines (rows for right side, columns for left)
  long long units;       // tiles * bands
  const void* coef;      // packed coefficient stream [bands][nblk][K+1][K]
  uint32_t* flags;       // [units] chunk-progress flags for in-place hand-offs
  void* trash;           // 32*R elements: write/read target of lanes past the last row
  int len;               // length of the rotated dimension (n right, m left)
  int k;                 // sweeps
  int bands;             // ceil(k / K)
  int nchunk;            // ceil(len / (K+1))
  int nblk;              // nchunk + 1
  int nw;                // warps per CTA
  int debug_no_chain;    // timing experiments only: every unit reads/writes A (wrong result)
  int debug_mode;        // timing experiments only (wrong result): 1 = no I/O or ring waits,
                         // 2 = no coefficient staging, 3 = both
  int smsp_group;        // place chain neighbours on the same SM sub-partition
  int elastic;           // rings only within a sub-partition group, flags across
};

// ------------------------------------------------------------------------------------
// one block of K+1 waves for one warp (fully unrolled; window slots are compile-time)
//   block b covers waves t = b(K+1)-1 .. b(K+1)+K-1. At the start of wave u it emits
//   column (b-1)(K+1)+u (finished after wave t-1) from slot u, then loads column
//   b(K+1)+u into slot u; lane l rotates columns (t-l, t-l+1) = slots (u-1-l, u-l).
// ------------------------------------------------------------------------------------
template <typename T, int K, int R, bool STRICT, bool REFL, bool EDGE, bool OUTRING>
__device__ __forceinline__ void run_block(T (&w)[R][K + 1], const Coef<T, REFL>* __restrict__ cb,
                                          const T* __restrict__ islot, T* __restrict__ oslot,
                                          T* const (&grow)[R], const long long (&gcs)[R],
                                          int b, int len, int Kb, int lane, bool has_in_rt, bool has_out_rt) {
  constexpr int TR = 32 * R;
  const long long c0 = (long long)b * (K + 1);
  // interior blocks always have input and output; only edge blocks test at run time
  const bool has_in = !EDGE || has_in_rt;
  const bool has_out = !EDGE || has_out_rt;
  // global output: one running pointer per row (rows past the matrix write a trash slot
  // with stride 0, so the store needs no predicate)
  T* gp[R];
  if constexpr (!OUTRING) {
#pragma unroll
    for (int r = 0; r < R; ++r) gp[r] = grow[r] + (c0 - (K + 1)) * gcs[r];
  }
#pragma unroll
  for (int u = 0; u <= K; ++u) {
    if (has_out) {
      const long long col = c0 - (K + 1) + u;
      if (!EDGE || col < len) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if constexpr (OUTRING) {
            oslot[u * TR + lane + 32 * r] = w[r][u];
          } else {
            *gp[r] = w[r][u];
          }
        }
      }
      if constexpr (!OUTRING) {
#pragma unroll
        for (int r = 0; r < R; ++r) gp[r] += gcs[r];
      }
    }
    {
      const long long col = c0 + u;
      if (!EDGE || (has_in && col < len)) {
#pragma unroll
        for (int r = 0; r < R; ++r) w[r][u] = islot[u * TR + lane + 32 * r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) w[r][u] = T(0);
      }
    }
#pragma unroll
    for (int l = 0; l < K; ++l) {
      constexpr int M = K + 1;
      const int sx = (u - 1 - l + 2 * M) % M;
      const int sy = (sx + 1) % M;
      if (EDGE) {
        const long long j = c0 + u - 1 - l;
        if (l >= Kb || j < 0 || j > (long long)len - 2) continue;
      }
      const Coef<T, REFL> cf = cb[u * K + l];
#pragma unroll
      for (int r = 0; r < R; ++r) xform<T, STRICT, REFL>(w[r][sx], w[r][sy], cf);
    }
  }
}

// ------------------------------------------------------------------------------------
// the persistent band-pipeline kernel
// ------------------------------------------------------------------------------------
template <typename T, int K, int R, bool STRICT, bool REFL>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) rs_pipeline_kernel(const __grid_constant__ PipeParams P) {
  using CoefT = Coef<T, REFL>;
  constexpr int TR = 32 * R;
  constexpr int CHUNK = (K + 1) * TR;  // elements of one ring chunk (K+1 columns x TR owners)
  constexpr int CBLK = (K + 1) * K;    // coefficient records per block
  constexpr int S = kStages;
  // per-warp control words: full[S] (mbarriers), consumed-chunk counter, coef[2] (mbarriers).
  // "full" is alias-safe as an mbarrier (the consumer has always seen chunk seq-S before it
  // waits for seq). "empty" is a monotonic counter instead: a ring's producer changes
  // between rounds (previous warp vs. self-fill), so a producer may have to wait on a
  // consumer many phases behind, which a parity test cannot express.
  constexpr int NBAR = kCtlWords;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int NW = P.nw;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long U = P.units;
  const long long G = gridDim.x;
  const long long ub = U * (long long)blockIdx.x / G;
  const long long ue = U * (long long)(blockIdx.x + 1) / G;
  // Position of this warp inside a round: chain neighbours (positions q, q+1) share an SM
  // sub-partition (warp id mod 4), and the positions used in the first round are balanced
  // over the four sub-partitions (10 units -> 3,3,2,2); idle warps take the rest.
  int qpos;
  {
    const int n_eff = (int)min((long long)NW, ue - ub);
    const int sub = warp & 3, idx = warp >> 2;
    int act_start = 0, idle_start = 0;
    for (int s2 = 0; s2 < sub; ++s2) {
      const int c = (n_eff - s2 + 3) / 4;
      act_start += c;
      idle_start += (NW - s2 + 3) / 4 - c;
    }
    const int c_sub = (n_eff - sub + 3) / 4;
    qpos = idx < c_sub ? act_start + idx : n_eff + idle_start + (idx - c_sub);
  }
  CoefT* coef_sm = reinterpret_cast<CoefT*>(smem_raw);
  T* ring_sm = reinterpret_cast<T*>(coef_sm + (size_t)NW * 2 * CBLK);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring_sm + (size_t)NW * S * CHUNK);

  if (threadIdx.x < NW) {
    uint64_t* bw = bars + threadIdx.x * NBAR;
#pragma unroll
    for (int i = 0; i < S; ++i) mbar_init(bw + i, 1);
    *reinterpret_cast<volatile uint32_t*>(bw + S) = 0u;
    mbar_init(bw + S + 1, 1);
    mbar_init(bw + S + 2, 1);
  }
  __syncthreads();

  T* const A = reinterpret_cast<T*>(P.A);
  const int len = P.len;
  const int nchunk = P.nchunk;
  const int nblk = P.nblk;
  const int bands = P.bands;
  uint64_t* const bar_in = bars + qpos * NBAR;  // full_in[S], consumed, coef[2]
  uint64_t* const full_in = bar_in;
  uint32_t* const consumed_in = reinterpret_cast<uint32_t*>(bar_in + S);
  uint64_t* const cbar = bar_in + S + 1;
  uint64_t* const full_out = bars + (qpos + 1) * NBAR;  // next position's ring (only with DST_RING)
  const uint32_t* const consumed_out = reinterpret_cast<const uint32_t*>(full_out + S);
  T* const rin = ring_sm + (size_t)qpos * S * CHUNK;
  T* const rout = ring_sm + (size_t)(qpos + 1) * S * CHUNK;
  CoefT* const cbuf = coef_sm + (size_t)qpos * 2 * CBLK;
  constexpr uint32_t kCoefBytes = (uint32_t)(CBLK * sizeof(CoefT));

  // Processing order inside the CTA: when the range ends in a partial tile (its low bands
  // feed the next CTA), run that tail first so the next CTA's start never waits for this
  // CTA's last round; the rest follows in natural tile-major order.
  const long long tail_start = (ue / bands) * bands;
  const bool reorder = (ue % bands != 0) && (tail_start > ub);
  const long long ntail = reorder ? ue - tail_start : 0;
  auto unit_at = [&](long long p) -> long long {
    return reorder ? (p < ntail ? tail_start + p : ub + (p - ntail)) : ub + p;
  };
  auto pos_of = [&](long long uu) -> long long {
    return reorder ? (uu >= tail_start ? uu - tail_start : uu - ub + ntail) : uu - ub;
  };

  uint32_t cseq = 0;  // coefficient blocks consumed by this warp (buffer = cseq&1)

  for (int jr = 0;; ++jr) {
    const long long p = (long long)jr * NW + qpos;
    if (p >= ue - ub) break;
    const long long u = unit_at(p);
    const long long tile = u / bands;
    const int band = (int)(u - tile * bands);
    const int Kb = min(K, P.k - band * K);
    // producer of u is u-1, consumer is u+1 (same tile); ring hand-off only when they are
    // adjacent positions of the same round of this CTA, else through A + progress flag.
    const int src = band == 0 ? SRC_GLOBAL
                              : ((qpos > 0 && u - 1 >= ub && pos_of(u - 1) == p - 1) ? SRC_RING : SRC_FLAG);
    const int dst = band == bands - 1
                        ? DST_GLOBAL
                        : ((qpos < NW - 1 && u + 1 < ue && pos_of(u + 1) == p + 1) ? DST_RING : DST_FLAG);
    const bool self = src != SRC_RING;

    T* grow[R];        // element (row r, column 0) of this lane's lines
    long long gcs[R];  // column stride; 0 for rows past the matrix (they use the trash slot)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long o = tile * TR + lane + 32 * r;
      const bool ok = o < P.owners;
      grow[r] = ok ? A + o * P.os : reinterpret_cast<T*>(P.trash) + lane + 32 * r;
      gcs[r] = ok ? P.cs : 0;
    }
    const CoefT* csrc = reinterpret_cast<const CoefT*>(P.coef) + (size_t)band * nblk * CBLK;
    const uint32_t seq0 = (uint32_t)jr * (uint32_t)nchunk;
    const uint32_t* myflag = P.flags + u;
    uint32_t* const outflag = P.flags + u + 1;

    // coefficient block 0 of this unit
    if (lane == 0) bulk_g2s(cbuf + (cseq & 1) * CBLK, csrc, kCoefBytes, &cbar[cseq & 1]);

    // self-filled input (band 0 reads A; a hand-off reads A after the producer's flag):
    // cp.async (LDGSTS) straight into this warp's own ring slot, two chunks ahead.
    uint32_t flag_seen = 0;
    auto fill_chunk = [&](int q) {
      if (src == SRC_FLAG && flag_seen < (uint32_t)q + 1) flag_seen = wait_flag(myflag, (uint32_t)q + 1);
      T* dstp = rin + ((seq0 + (uint32_t)q) % S) * CHUNK;
      const long long c0 = (long long)q * (K + 1);
      const T* sp[R];
#pragma unroll
      for (int r = 0; r < R; ++r) sp[r] = grow[r] + c0 * gcs[r];
      if (c0 + K < len) {
#pragma unroll
        for (int v = 0; v <= K; ++v) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            cp_async_elem(dstp + v * TR + lane + 32 * r, sp[r], true);
            sp[r] += gcs[r];
          }
        }
      } else {
#pragma unroll
        for (int v = 0; v <= K; ++v) {
          const bool cv = c0 + v < len;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            cp_async_elem(dstp + v * TR + lane + 32 * r, cv ? sp[r] : grow[r], cv);
            sp[r] += gcs[r];
          }
        }
      }
      cp_async_commit();
    };
    // Self-filled chunks still arrive on full_in (nobody waits on them) so the barrier's
    // phase count stays equal to the chunk sequence number for ring-fed rounds later on.
    if (self) {
      fill_chunk(0);
      if (1 < nchunk) fill_chunk(1);
      if (1 < nchunk)
        cp_async_wait_group<1>();
      else
        cp_async_wait_group<0>();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_in[seq0 % S]);
    }

    T w[R][K + 1];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int s = 0; s <= K; ++s) w[r][s] = T(0);

    const int full_hi = (Kb == K && len - 1 - K >= 0) ? (len - 1 - K) / (K + 1) : 0;

    // One block: protocol + compute. EDGE / OUTRING are compile-time so the interior loop
    // carries no per-block branches beyond the hand-off protocol of this unit.
    auto block = [&](int b, auto edge_c, auto outring_c) {
      constexpr bool EDGE = decltype(edge_c)::value;
      constexpr bool OUTRING = decltype(outring_c)::value;
      if (lane == 0 && b + 1 < nblk)
        bulk_g2s(cbuf + ((cseq + 1) & 1) * CBLK, csrc + (size_t)(b + 1) * CBLK, kCoefBytes, &cbar[(cseq + 1) & 1]);
      const bool has_in = !EDGE || b < nchunk;
      const bool has_out = !EDGE || b >= 1;
      if (self && b + 2 < nchunk) fill_chunk(b + 2);
      const uint32_t iseq = seq0 + (uint32_t)b;
      const T* islot = rin + (iseq % S) * CHUNK;
      const uint32_t oseq = seq0 + (uint32_t)b - 1u;
      T* oslot = rout + (oseq % S) * CHUNK;
      mbar_wait(&cbar[cseq & 1], (cseq >> 1) & 1u);
      if (!self && has_in) mbar_wait(&full_in[iseq % S], (iseq / S) & 1u);
      if (OUTRING && has_out && oseq >= (uint32_t)S) wait_count(consumed_out, oseq - S + 1u);
      run_block<T, K, R, STRICT, REFL, EDGE, OUTRING>(w, cbuf + (cseq & 1) * CBLK, islot, oslot, grow, gcs, b, len,
                                                      Kb, lane, b < nchunk, b >= 1);
      __syncwarp();
      if (lane == 0) {
        if (has_in) st_release_shared(consumed_in, iseq + 1u);
        if (OUTRING && has_out) mbar_arrive(&full_out[oseq % S]);
        if (dst == DST_FLAG && has_out && ((b & (kFlagEvery - 1)) == 0 || b == nblk - 1)) {
          // the warp barrier above orders every lane's stores before lane 0's gpu-scope
          // fence; the release store then publishes "chunks 0..b-1 are in A"
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          st_release(outflag, (uint32_t)b);
        }
      }
      if (self && b + 1 < nchunk) {  // the chunk read by the next block has landed
        if (b + 2 < nchunk)
          cp_async_wait_group<1>();
        else
          cp_async_wait_group<0>();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_in[(iseq + 1u) % S]);
      }
      ++cseq;
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    const int interior_end = full_hi + 1;  // blocks [1, full_hi] are interior
    if (dst == DST_RING) {
      block(0, T_{}, T_{});
      for (int b = 1; b < interior_end; ++b) block(b, F_{}, T_{});
      for (int b = max(1, interior_end); b < nblk; ++b) block(b, T_{}, T_{});
    } else {
      block(0, T_{}, F_{});
      for (int b = 1; b < interior_end; ++b) block(b, F_{}, F_{});
      for (int b = max(1, interior_end); b < nblk; ++b) block(b, T_{}, F_{});
    }
  }
}

// ------------------------------------------------------------------------------------
// v2: lock-step band groups inside a warp ("group pipeline")
//   A warp runs G consecutive bands of one tile of TR = (32/G)*R owners: lane group g
//   (lanes g*32/G ..) applies band bg*G+g to the same TR rows. Group g processes block
//   b-g at step b, so the column group g emits at wave u is exactly the column group g+1
//   loads at the same wave: it moves with shfl.up (no waiting, no shared memory). Only
//   group 0's input and group G-1's output go through rings / A, so a tile's chain has
//   bands/G - 1 inter-warp links instead of bands - 1.
// ------------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T shfl_up_t(T v, int d) {
  return __shfl_up_sync(0xffffffffu, v, d);
}

template <typename T, int K, int R, int G, bool STRICT, bool REFL, bool EDGE, bool OUTRING>
__device__ __forceinline__ void gp_step(T (&w)[R][K + 1], const Coef<T, REFL>* __restrict__ cb,
                                        const T* __restrict__ islot, T* __restrict__ oslot,
                                        T* const (&gout)[R], const long long (&gcs)[R], int b, int len, int nblk,
                                        int grp, int Kb, int sl, bool in_ok, bool out_ok) {
  constexpr int LPG = 32 / G;
  constexpr int TR = LPG * R;
  const int gb = b - grp;  // this lane group's block
  const bool gact = !EDGE || (gb >= 0 && gb < nblk);
  const long long c0 = (long long)gb * (K + 1);
  const long long ic0 = (long long)b * (K + 1);        // group 0's input columns
  const long long oc0 = (long long)(b - G) * (K + 1);  // group G-1's output columns
  const bool last = grp == G - 1;
  const bool first = grp == 0;
  T* gp[R];
  if constexpr (!OUTRING) {
#pragma unroll
    for (int r = 0; r < R; ++r) gp[r] = gout[r] + oc0 * gcs[r];
  }
#pragma unroll
  for (int u = 0; u <= K; ++u) {
    T e[R];
#pragma unroll
    for (int r = 0; r < R; ++r) e[r] = w[r][u];
    // group G-1 emits column (b-G)(K+1)+u to the next warp / A
    if (last && (!EDGE || (out_ok && oc0 + u < len))) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (OUTRING)
          oslot[u * TR + sl + LPG * r] = e[r];
        else
          *gp[r] = e[r];
      }
    }
    if constexpr (!OUTRING) {
#pragma unroll
      for (int r = 0; r < R; ++r) gp[r] += gcs[r];
    }
    // group g > 0 takes group g-1's emitted column; group 0 reads the ring
    T v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = shfl_up_t(e[r], LPG);
    if (first) {
      if (!EDGE || (in_ok && ic0 + u < len)) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = islot[u * TR + sl + LPG * r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = T(0);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) w[r][u] = v[r];
#pragma unroll
    for (int l = 0; l < K; ++l) {
      constexpr int M = K + 1;
      const int sx = (u - 1 - l + 2 * M) % M;
      const int sy = (sx + 1) % M;
      const Coef<T, REFL> cf = cb[(u * K + l) * G];
      if constexpr (EDGE) {
        const long long j = c0 + u - 1 - l;
        const bool valid = gact && l < Kb && j >= 0 && j <= (long long)len - 2;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          T x = w[r][sx], y = w[r][sy];
          xform<T, STRICT, REFL>(x, y, cf);
          w[r][sx] = valid ? x : w[r][sx];
          w[r][sy] = valid ? y : w[r][sy];
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) xform<T, STRICT, REFL>(w[r][sx], w[r][sy], cf);
      }
    }
  }
}

template <typename T, int K, int R, int G, bool STRICT, bool REFL>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) rs_gpipe_kernel(const __grid_constant__ PipeParams P) {
  using CoefT = Coef<T, REFL>;
  constexpr int LPG = 32 / G;
  constexpr int TR = LPG * R;          // owners per tile
  constexpr int CHUNK = (K + 1) * TR;  // ring chunk: K+1 columns x TR owners
  constexpr int CBLK = (K + 1) * K;
  constexpr int S = kStages;
  constexpr int NBAR = kCtlWords;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int NW = P.nw;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPG;
  const int sl = lane - grp * LPG;
  CoefT* coef_sm = reinterpret_cast<CoefT*>(smem_raw);                       // [NW][2][G][CBLK]
  T* ring_sm = reinterpret_cast<T*>(coef_sm + (size_t)NW * 2 * G * CBLK);   // [NW][S][CHUNK]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring_sm + (size_t)NW * S * CHUNK);
  if (threadIdx.x < NW) {
    uint64_t* bw = bars + threadIdx.x * NBAR;
#pragma unroll
    for (int i = 0; i < S; ++i) mbar_init(bw + i, 1);
    *reinterpret_cast<volatile uint32_t*>(bw + S) = 0u;
    mbar_init(bw + S + 1, 1);
    mbar_init(bw + S + 2, 1);
  }
  __syncthreads();

  const long long U = P.units;
  const long long Gr = gridDim.x;
  const long long ub = U * (long long)blockIdx.x / Gr;
  const long long ue = U * (long long)(blockIdx.x + 1) / Gr;
  // chain neighbours on the same SM sub-partition, balanced over the four (see v1)
  int qpos = warp;
  {
    const int n_eff = (int)min((long long)NW, ue - ub);
    const int sub = warp & 3, idx = warp >> 2;
    int act_start = 0, idle_start = 0;
    for (int s2 = 0; s2 < sub; ++s2) {
      const int c = (n_eff - s2 + 3) / 4;
      act_start += c;
      idle_start += (NW - s2 + 3) / 4 - c;
    }
    const int c_sub = (n_eff - sub + 3) / 4;
    qpos = idx < c_sub ? act_start + idx : n_eff + idle_start + (idx - c_sub);
  }

  T* const A = reinterpret_cast<T*>(P.A);
  const int len = P.len;
  const int nchunk = P.nchunk;
  const int nblk = P.nblk;
  const int nsteps = nblk + G - 1;
  const int bgroups = (P.bands + G - 1) / G;
  uint64_t* const bar_in = bars + qpos * NBAR;
  uint64_t* const full_in = bar_in;
  uint32_t* const consumed_in = reinterpret_cast<uint32_t*>(bar_in + S);
  uint64_t* const cbar = bar_in + S + 1;
  uint64_t* const full_out = bars + (qpos + 1) * NBAR;
  const uint32_t* const consumed_out = reinterpret_cast<const uint32_t*>(full_out + S);
  T* const rin = ring_sm + (size_t)qpos * S * CHUNK;
  T* const rout = ring_sm + (size_t)(qpos + 1) * S * CHUNK;
  CoefT* const cbuf = coef_sm + (size_t)qpos * 2 * G * CBLK;
  constexpr uint32_t kCoefBytes = (uint32_t)(CBLK * sizeof(CoefT));

  const long long tail_start = (ue / bgroups) * bgroups;
  const bool reorder = (ue % bgroups != 0) && (tail_start > ub);
  const long long ntail = reorder ? ue - tail_start : 0;
  auto unit_at = [&](long long p) -> long long {
    return reorder ? (p < ntail ? tail_start + p : ub + (p - ntail)) : ub + p;
  };
  auto pos_of = [&](long long uu) -> long long {
    return reorder ? (uu >= tail_start ? uu - tail_start : uu - ub + ntail) : uu - ub;
  };

  uint32_t cseq = 0;
  for (int jr = 0;; ++jr) {
    const long long p = (long long)jr * NW + qpos;
    if (p >= ue - ub) break;
    const long long u = unit_at(p);
    const long long tile = u / bgroups;
    const int bgi = (int)(u - tile * bgroups);
    const int band0 = bgi * G;
    const int myband = band0 + grp;
    const int Kb = myband < P.bands ? min(K, P.k - myband * K) : 0;
    int src = bgi == 0 ? SRC_GLOBAL : ((qpos > 0 && u - 1 >= ub && pos_of(u - 1) == p - 1) ? SRC_RING : SRC_FLAG);
    int dst = bgi == bgroups - 1 ? DST_GLOBAL
                                 : ((qpos < NW - 1 && u + 1 < ue && pos_of(u + 1) == p + 1) ? DST_RING : DST_FLAG);
    // every group is a full band of K sweeps and every band exists -> interior steps allowed
    const bool all_full = (band0 + G <= P.bands) && (P.k - (band0 + G - 1) * K >= K);

    // per-lane row pointers: group 0 lanes read A (self-fill), group G-1 lanes write A
    T* grow[R];
    long long gcs[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long o = tile * TR + sl + LPG * r;
      const bool ok = o < P.owners;
      grow[r] = ok ? A + o * P.os : reinterpret_cast<T*>(P.trash) + lane + 32 * r;
      gcs[r] = ok ? P.cs : 0;
    }
    const uint32_t seq0 = (uint32_t)jr * (uint32_t)nchunk;
    const uint32_t* myflag = P.flags + u;

    const int nsteps_pack = nblk + G - 1;
    const CoefT* csrc = reinterpret_cast<const CoefT*>(P.coef) + (size_t)bgi * nsteps_pack * G * CBLK;
    auto issue_coef = [&](int step, uint32_t buf) {
      if (lane == 0)
        bulk_g2s(cbuf + (size_t)buf * G * CBLK, csrc + (size_t)step * G * CBLK, G * kCoefBytes, &cbar[buf]);
    };
    issue_coef(0, cseq & 1);

    uint32_t flag_seen = 0;
    auto fill_chunk = [&](int q) {
      if (src == SRC_FLAG && flag_seen < (uint32_t)q + 1) flag_seen = wait_flag(myflag, (uint32_t)q + 1);
      T* dstp = rin + ((seq0 + (uint32_t)q) % S) * CHUNK;
      if (grp == 0) {
        const long long c0 = (long long)q * (K + 1);
        const T* sp[R];
#pragma unroll
        for (int r = 0; r < R; ++r) sp[r] = grow[r] + c0 * gcs[r];
#pragma unroll
        for (int v = 0; v <= K; ++v) {
          const bool cv = c0 + v < len;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            cp_async_elem(dstp + v * TR + sl + LPG * r, cv ? sp[r] : grow[r], cv);
            sp[r] += gcs[r];
          }
        }
      }
      cp_async_commit();
    };
    auto publish_chunk = [&](int q, bool younger_in_flight) {
      if (younger_in_flight)
        cp_async_wait_group<1>();
      else
        cp_async_wait_group<0>();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_in[(seq0 + (uint32_t)q) % S]);
    };
    if (src != SRC_RING) {
      fill_chunk(0);
      if (1 < nchunk) fill_chunk(1);
      publish_chunk(0, 1 < nchunk);
    }

    T w[R][K + 1];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int s2 = 0; s2 <= K; ++s2) w[r][s2] = T(0);

    const int full_hi = (len - 1 - K >= 0) ? (len - 1 - K) / (K + 1) : 0;

    for (int b = 0; b < nsteps; ++b) {
      if (b + 1 < nsteps) issue_coef(b + 1, (cseq + 1) & 1);
      const bool self_next = (src != SRC_RING) && (b + 1 < nchunk);
      const bool self_next2 = (src != SRC_RING) && (b + 2 < nchunk);
      if (self_next2) fill_chunk(b + 2);

      mbar_wait(&cbar[cseq & 1], (cseq >> 1) & 1u);
      const bool in_ok = b < nchunk;
      const int oq = b - G;  // output chunk of this step
      const bool out_ok = oq >= 0 && oq < nchunk;
      const uint32_t iseq = seq0 + (uint32_t)b;
      const T* islot = rin + (iseq % S) * CHUNK;
      if (in_ok) mbar_wait(&full_in[iseq % S], (iseq / S) & 1u);
      const uint32_t oseq = seq0 + (uint32_t)oq;
      T* oslot = rout + (oseq % S) * CHUNK;
      if (dst == DST_RING && out_ok && oseq >= (uint32_t)S) wait_count(consumed_out, oseq - S + 1u);

      const CoefT* cb = cbuf + (size_t)(cseq & 1) * G * CBLK + grp;  // record (u,l) at cb[(u*K+l)*G]
      const bool interior = all_full && b >= G && b <= full_hi;
      if (interior) {
        if (dst == DST_RING)
          gp_step<T, K, R, G, STRICT, REFL, false, true>(w, cb, islot, oslot, grow, gcs, b, len, nblk, grp, Kb, sl,
                                                          in_ok, out_ok);
        else
          gp_step<T, K, R, G, STRICT, REFL, false, false>(w, cb, islot, oslot, grow, gcs, b, len, nblk, grp, Kb, sl,
                                                           in_ok, out_ok);
      } else {
        if (dst == DST_RING)
          gp_step<T, K, R, G, STRICT, REFL, true, true>(w, cb, islot, oslot, grow, gcs, b, len, nblk, grp, Kb, sl,
                                                         in_ok, out_ok);
        else
          gp_step<T, K, R, G, STRICT, REFL, true, false>(w, cb, islot, oslot, grow, gcs, b, len, nblk, grp, Kb, sl,
                                                          in_ok, out_ok);
      }
      __syncwarp();
      if (lane == 0) {
        if (in_ok) st_release_shared(consumed_in, iseq + 1u);
        if (dst == DST_RING && out_ok) mbar_arrive(&full_out[oseq % S]);
      }
      if (dst == DST_FLAG && out_ok && lane == 0 && ((oq & (kFlagEvery - 1)) == 0 || oq == nchunk - 1)) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        st_release(P.flags + u + 1, (uint32_t)(oq + 1));
      }
      if (self_next) publish_chunk(b + 1, self_next2);
      ++cseq;
    }
  }
}

// ------------------------------------------------------------------------------------
// coefficient repack: C/S (len-1) x k column-major -> [bands][nblk][K+1][K] records.
// Entry (band, b, u, l) holds sweep p = band*K + l, rotation j = b(K+1)+u-1-l, or zeros
// when that lane is idle (startup/shutdown triangles, partial last band). Reverse order
// mirrors j and negates S (rotation) or C (reflector): both exact in IEEE arithmetic.
// ------------------------------------------------------------------------------------
template <typename T, int K, bool REFL>
__global__ void __launch_bounds__(256) rs_pack_kernel(Coef<T, REFL>* __restrict__ out, const T* __restrict__ C,
                                                      const T* __restrict__ Sm, long long ldcs, int len, int k,
                                                      int nblk, int rev) {
  // grid.y = band; consecutive threads write consecutive records (coalesced), and each
  // warp reads 8 coefficient columns x 4 consecutive rows (one sector per column)
  constexpr int E = (K + 1) * K;
  const int band = blockIdx.y;
  const int total = nblk * E;
  Coef<T, REFL>* dst = out + (size_t)band * total;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int b = i / E;
    const int e = i - b * E;
    const int u = e / K;
    const int l = e - u * K;
    const int p = band * K + l;
    const int j = b * (K + 1) + u - 1 - l;
    Coef<T, REFL> cf;
    if (p < k && j >= 0 && j <= len - 2) {
      const long long jj = rev ? (long long)(len - 2 - j) : (long long)j;
      T c = __ldg(C + jj + (long long)p * ldcs);
      T s = __ldg(Sm + jj + (long long)p * ldcs);
      if constexpr (REFL) {
        if (rev) c = -c;
        cf.s = s;
        cf.d = c - s;
        cf.e = c + s;
        cf.pad = T(0);
      } else {
        if (rev) s = -s;
        cf.c = c;
        cf.s = s;
      }
    } else {
      if constexpr (REFL) {
        cf.s = T(0);
        cf.d = T(0);
        cf.e = T(0);
        cf.pad = T(0);
      } else {
        cf.c = T(0);
        cf.s = T(0);
      }
    }
    dst[i] = cf;
  }
}

// Group-pipeline layout: [band group][step][u][l][g] — at step b lane group g needs block
// b-g of band bg*G+g, so one contiguous bulk copy per step serves all groups and the G
// records a warp reads for (u, l) are adjacent (one 16*G-byte segment per LDS.128).
template <typename T, int K, int G, bool REFL>
__global__ void __launch_bounds__(256) rs_pack_g_kernel(Coef<T, REFL>* __restrict__ out, const T* __restrict__ C,
                                                        const T* __restrict__ Sm, long long ldcs, int len, int k,
                                                        int bands, int nblk, int rev) {
  constexpr int E = (K + 1) * K * G;
  const int bg = blockIdx.y;
  const int nsteps = nblk + G - 1;
  const int total = nsteps * E;
  Coef<T, REFL>* dst = out + (size_t)bg * total;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int step = i / E;
    int e = i - step * E;
    const int u = e / (K * G);
    e -= u * (K * G);
    const int l = e / G;
    const int g = e - l * G;
    const int band = bg * G + g;
    const int blk = step - g;
    const int p = band * K + l;
    const int j = blk * (K + 1) + u - 1 - l;
    Coef<T, REFL> cf;
    if (band < bands && blk >= 0 && blk < nblk && p < k && j >= 0 && j <= len - 2) {
      const long long jj = rev ? (long long)(len - 2 - j) : (long long)j;
      T c = __ldg(C + jj + (long long)p * ldcs);
      T s = __ldg(Sm + jj + (long long)p * ldcs);
      if constexpr (REFL) {
        if (rev) c = -c;
        cf.s = s;
        cf.d = c - s;
        cf.e = c + s;
        cf.pad = T(0);
      } else {
        if (rev) s = -s;
        cf.c = c;
        cf.s = s;
      }
    } else {
      if constexpr (REFL) {
        cf.s = T(0);
        cf.d = T(0);
        cf.e = T(0);
        cf.pad = T(0);
      } else {
        cf.c = T(0);
        cf.s = T(0);
      }
    }
    dst[i] = cf;
  }
}

// ------------------------------------------------------------------------------------
// naive kernel: one thread per owner, plain sweep loop (GPU restatement of _naive_py,
// core.py:195-205); independent second implementation used for cross-checks.
// ------------------------------------------------------------------------------------
template <typename T, bool STRICT, bool REFL>
__global__ void rs_naive_kernel(T* __restrict__ A, long long os, long long cs, long long owners, int len,
                                const T* __restrict__ C, const T* __restrict__ Sm, long long ldcs, int k, int rev) {
  const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (o >= owners) return;
  T* a = A + o * os;
  for (int p = 0; p < k; ++p) {
    for (int jj = 0; jj < len - 1; ++jj) {
      const long long j = rev ? (long long)len - 2 - jj : jj;
      const T c = C[j + (long long)p * ldcs];
      const T s = Sm[j + (long long)p * ldcs];
      T x = a[j * cs];
      T y = a[(j + 1) * cs];
      if constexpr (REFL) {
        const T d = sub_rn(c, s);
        const T e = add_rn(c, s);
        refl2<T, STRICT>(x, y, s, d, e);
      } else {
        rot2<T, STRICT>(x, y, c, s);
      }
      a[j * cs] = x;
      a[(j + 1) * cs] = y;
    }
  }
}

// ------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------
struct Geometry {
  long long owners = 0;
  int len = 0;
  long long os = 0, cs = 0;
  int k = 0;
  int bands = 0;
  long long tiles = 0;
  long long units = 0;
  int nchunk = 0;
  int nblk = 0;
  size_t coef_bytes = 0;
  size_t flag_bytes = 0;
  size_t coef_rec = 0;
  long long units_g2 = 0;  // v2 group pipeline, G = 2 (tiles of 32 owners)
  long long units_g4 = 0;  // v2 group pipeline, G = 4 (tiles of 16 owners)
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

bool make_geometry(int64_t m, int64_t n, int64_t lda, int64_t k, int side, int kind, int dtype, Geometry* g) {
  const bool left = side == RS_SIDE_LEFT;
  g->owners = left ? n : m;
  g->len = (int)(left ? m : n);
  g->os = left ? lda : 1;
  g->cs = left ? 1 : lda;
  g->k = (int)k;
  g->bands = (int)((k + kK - 1) / kK);
  g->tiles = (g->owners + kTileOwners - 1) / kTileOwners;
  g->units = g->tiles * g->bands;
  g->nchunk = (g->len + kK) / (kK + 1);
  g->nblk = g->nchunk + 1;
  const size_t tsz = dtype == RS_DTYPE_F64 ? 8 : 4;
  g->coef_rec = (kind == RS_KIND_REFLECTOR ? 4 : 2) * tsz;
  {
    const size_t per_rec = (size_t)(kK + 1) * kK * g->coef_rec;
    size_t v1 = (size_t)g->bands * g->nblk * per_rec;
    size_t g2 = (size_t)((g->bands + 1) / 2) * (g->nblk + 1) * 2 * per_rec;
    size_t g4 = (size_t)((g->bands + 3) / 4) * (g->nblk + 3) * 4 * per_rec;
    size_t mx = v1 > g2 ? v1 : g2;
    if (g4 > mx) mx = g4;
    g->coef_bytes = align_up(mx, 256);
  }
  g->units_g2 = ((g->owners + 16 * kR - 1) / (16 * kR)) * ((g->bands + 1) / 2);
  g->units_g4 = ((g->owners + 8 * kR - 1) / (8 * kR)) * ((g->bands + 3) / 4);
  long long umax = g->units;
  if (g->units_g2 > umax) umax = g->units_g2;
  if (g->units_g4 > umax) umax = g->units_g4;
  g->flag_bytes = align_up((size_t)(umax + 1) * sizeof(uint32_t), 256) + kTrashBytes;
  return true;
}

struct LaunchPlan {
  int grid = 0;
  int nw = 0;
  size_t smem = 0;
  long long units = 0;
  int variant = 0;
};

// kernel variants: v1 = one band per warp; g2 / g4 = lock-step groups of 2 / 4 bands
enum : int { VAR_V1 = 0, VAR_G2 = 2, VAR_G4 = 4 };

int kernel_variant() {
  const char* e = getenv("RS_KERNEL");
  if (e == nullptr) return VAR_V1;
  if (strcmp(e, "v1") == 0) return VAR_V1;
  if (strcmp(e, "g2") == 0) return VAR_G2;
  return VAR_G4;
}

size_t smem_per_warp(size_t tsz, size_t coef_rec, int variant) {
  const size_t cblk = (size_t)(kK + 1) * kK * coef_rec;
  if (variant == VAR_V1)
    return 2 * cblk + (size_t)kStages * (kK + 1) * kTileOwners * tsz + kCtlWords * sizeof(uint64_t);
  const size_t groups = (size_t)variant;
  const size_t tile = (size_t)(32 / variant) * kR;
  return 2 * groups * cblk + (size_t)kStages * (kK + 1) * tile * tsz + kCtlWords * sizeof(uint64_t);
}

long long variant_units(const Geometry& g, int variant) {
  return variant == VAR_V1 ? g.units : (variant == VAR_G2 ? g.units_g2 : g.units_g4);
}

rs_status plan_launch(const Geometry& g, size_t tsz, int variant, LaunchPlan* lp) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(RS_ECUDA, "cudaGetDevice failed");
  int sms = 0, optin = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return fail(RS_ECUDA, "cudaDeviceGetAttribute failed");
  const size_t per = smem_per_warp(tsz, g.coef_rec, variant);
  const long long units = variant_units(g, variant);
  // one extra control block for the (never used) ring of warp nw
  int cap = (int)((optin - kCtlWords * sizeof(uint64_t)) / per);
  if (cap > kMaxWarps) cap = kMaxWarps;
  if (cap < 1) return fail(RS_EUNSUPPORTED, "shared memory too small for one pipeline warp");
  long long grid = sms;
  // test hooks: force multi-round / multi-CTA geometry on small problems
  if (const char* ev = getenv("RS_DEBUG_MAX_WARPS")) {
    const int v = atoi(ev);
    if (v >= 1 && v < cap) cap = v;
  }
  if (const char* ev = getenv("RS_DEBUG_GRID")) {
    const long long v = atoll(ev);
    if (v >= 1 && v < grid) grid = v;
  }
  if (units < grid) grid = units;
  if (grid < 1) grid = 1;
  const double x = (double)units / (double)grid;
  // units per CTA x: one round of ceil(x) warps when it fits, else the fewest rounds of
  // at most `cap` warps, spread evenly so the last round is as full as possible.
  long long rounds = (long long)ceil(x / cap);
  if (rounds < 1) rounds = 1;
  int nw = (int)ceil(x / (double)rounds);
  if (nw > cap) nw = cap;
  if (nw < 1) nw = 1;
  // Multi-round CTAs: a warp count that is a multiple of 4 keeps the four SM
  // sub-partitions equally loaded (measured: 12 warps beat 14 by ~6% on config 3), when the
  // CTA runs many rounds anyway (few-round CTAs lose more to the extra round: config 5).
  if (rounds >= 4 && (nw & 3) != 0 && nw > 4) {
    const int nw4 = nw & ~3;
    const long long r4 = (long long)ceil(x / nw4);
    if (4 * r4 <= 5 * rounds + 4) nw = nw4;
  }
  lp->grid = (int)grid;
  lp->nw = nw;
  lp->smem = per * nw + kCtlWords * sizeof(uint64_t);
  lp->units = units;
  lp->variant = variant;
  return RS_OK;
}

template <typename T, bool REFL>
rs_status launch_pack(const Geometry& g, const T* C, const T* S, long long ldcs, int rev, void* ws,
                      cudaStream_t st) {
  using CoefT = Coef<T, REFL>;
  CoefT* coef = reinterpret_cast<CoefT*>(ws);
  const int variant = kernel_variant();
  if (variant == VAR_V1) {
    const int per_band = g.nblk * (kK + 1) * kK;
    int bx = (per_band + 255) / 256;
    if (bx > 64) bx = 64;
    dim3 pgrid((unsigned)bx, (unsigned)g.bands);
    rs_pack_kernel<T, kK, REFL><<<pgrid, 256, 0, st>>>(coef, C, S, ldcs, g.len, g.k, g.nblk, rev);
  } else {
    const int G = variant;
    const int per_group = (g.nblk + G - 1) * (kK + 1) * kK * G;
    int bx = (per_group + 255) / 256;
    if (bx > 128) bx = 128;
    dim3 pgrid((unsigned)bx, (unsigned)((g.bands + G - 1) / G));
    if (G == 2)
      rs_pack_g_kernel<T, kK, 2, REFL><<<pgrid, 256, 0, st>>>(coef, C, S, ldcs, g.len, g.k, g.bands, g.nblk, rev);
    else
      rs_pack_g_kernel<T, kK, 4, REFL><<<pgrid, 256, 0, st>>>(coef, C, S, ldcs, g.len, g.k, g.bands, g.nblk, rev);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("pack launch: ") + cudaGetErrorString(e));
  return RS_OK;
}

// Runs the pipeline on coefficients already packed into `ws` (by launch_pack with the
// same geometry, order and kind). Resets the hand-off flags first.
template <typename T, bool STRICT, bool REFL>
rs_status launch_run(const Geometry& g, T* Abase, int rev, void* ws, cudaStream_t st) {
  using CoefT = Coef<T, REFL>;
  LaunchPlan lp;
  rs_status rc = plan_launch(g, sizeof(T), kernel_variant(), &lp);
  if (rc != RS_OK) return rc;
  CoefT* coef = reinterpret_cast<CoefT*>(ws);
  uint32_t* flags = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(ws) + g.coef_bytes);
  cudaError_t e = cudaMemsetAsync(flags, 0, g.flag_bytes - kTrashBytes, st);
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  PipeParams P;
  P.A = Abase;
  P.os = g.os;
  P.cs = rev ? -g.cs : g.cs;
  if (rev) P.A = Abase + (long long)(g.len - 1) * g.cs;
  P.owners = g.owners;
  P.units = lp.units;
  P.coef = coef;
  P.flags = flags;
  P.trash = reinterpret_cast<unsigned char*>(ws) + g.coef_bytes + g.flag_bytes - kTrashBytes;
  P.len = g.len;
  P.k = g.k;
  P.bands = g.bands;
  P.nchunk = g.nchunk;
  P.nblk = g.nblk;
  P.nw = lp.nw;
  P.debug_no_chain = getenv("RS_DEBUG_NO_CHAIN") ? atoi(getenv("RS_DEBUG_NO_CHAIN")) : 0;
  P.debug_mode = getenv("RS_DEBUG_MODE") ? atoi(getenv("RS_DEBUG_MODE")) : 0;
  P.smsp_group = getenv("RS_SMSP_GROUP") ? atoi(getenv("RS_SMSP_GROUP")) : 1;
  P.elastic = getenv("RS_ELASTIC") ? atoi(getenv("RS_ELASTIC")) : 0;
  auto kern = lp.variant == VAR_V1   ? rs_pipeline_kernel<T, kK, kR, STRICT, REFL>
              : lp.variant == VAR_G2 ? rs_gpipe_kernel<T, kK, kR, 2, STRICT, REFL>
                                     : rs_gpipe_kernel<T, kK, kR, 4, STRICT, REFL>;
  {
    // opt in to the large dynamic shared memory once per (kernel, device)
    static std::atomic<int> configured_mask[3] = {{0}, {0}, {0}};
    std::atomic<int>& configured = configured_mask[lp.variant == VAR_V1 ? 0 : (lp.variant == VAR_G2 ? 1 : 2)];
    int dev = 0;
    cudaGetDevice(&dev);
    const int bit = 1 << (dev & 31);
    if (!(configured.load(std::memory_order_relaxed) & bit)) {
      int optin = 0;
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      if (e != cudaSuccess) return fail(RS_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      configured.fetch_or(bit, std::memory_order_relaxed);
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)lp.grid);
  cfg.blockDim = dim3((unsigned)(lp.nw * 32));
  cfg.dynamicSmemBytes = lp.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, P);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("pipeline launch: ") + cudaGetErrorString(e));
  return RS_OK;
}

template <typename T, bool STRICT, bool REFL>
rs_status launch_naive(const Geometry& g, T* A, const T* C, const T* S, long long ldcs, int rev, cudaStream_t st) {
  const long long blocks = (g.owners + 127) / 128;
  rs_naive_kernel<T, STRICT, REFL><<<(unsigned)blocks, 128, 0, st>>>(A, g.os, g.cs, g.owners, g.len, C, S, ldcs,
                                                                       g.k, rev);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("naive launch: ") + cudaGetErrorString(e));
  return RS_OK;
}

template <typename T>
rs_status run_dispatch(const Geometry& g, T* A, int rev, int kind, int strict, void* ws, cudaStream_t st) {
  if (strict)
    return kind == RS_KIND_REFLECTOR ? launch_run<T, true, true>(g, A, rev, ws, st)
                                     : launch_run<T, true, false>(g, A, rev, ws, st);
  return kind == RS_KIND_REFLECTOR ? launch_run<T, false, true>(g, A, rev, ws, st)
                                   : launch_run<T, false, false>(g, A, rev, ws, st);
}

// Shared argument validation (reference: require_colmajor core.py:41-51, _check_apply_args
// core.py:110-117). Returns RS_OK and fills g, or an error.
rs_status validate(int64_t m, int64_t n, int64_t lda, int64_t ldcs, int64_t k, int side, int order, int kind,
                   int dtype, bool need_ldcs, Geometry* g) {
  if (side != RS_SIDE_RIGHT && side != RS_SIDE_LEFT) return fail(RS_EINVAL, "side must be 0 (right) or 1 (left)");
  if (order != RS_ORDER_FORWARD && order != RS_ORDER_REVERSE)
    return fail(RS_EINVAL, "order must be 0 (forward) or 1 (reverse)");
  if (kind != RS_KIND_ROTATION && kind != RS_KIND_REFLECTOR)
    return fail(RS_EINVAL, "kind must be 0 (rotation) or 1 (reflector)");
  if (m < 0 || n < 0) return fail(RS_EINVAL, "matrix dimensions must be non-negative");
  const bool left = side == RS_SIDE_LEFT;
  const int64_t len = left ? m : n;
  if (len < 2)
    return fail(RS_EINVAL, left ? "matrix needs at least 2 rows for left-side application"
                                : "matrix needs at least 2 columns");
  if (len > (int64_t)1 << 26) return fail(RS_EUNSUPPORTED, "rotated dimension longer than 2^26");
  if (k < 1) return fail(RS_EINVAL, "need k >= 1 sequences");
  if (k > (int64_t)65535 * kK) return fail(RS_EUNSUPPORTED, "more than 65535*8 sequences");
  if (lda < (m > 1 ? m : 1)) return fail(RS_EINVAL, "lda must be >= max(1, m) (column-major)");
  if (need_ldcs && ldcs < len - 1) return fail(RS_EINVAL, "ldcs must be >= len - 1");
  make_geometry(m, n, lda, k, side, kind, dtype, g);
  return RS_OK;
}

rs_status check_workspace(const Geometry& g, void* ws, size_t bytes) {
  if (ws == nullptr) return fail(RS_EINVAL, "packed mode needs a caller workspace");
  if (bytes < g.coef_bytes + g.flag_bytes) return fail(RS_ENOMEM, "workspace smaller than rs_workspace_bytes()");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(RS_EINVAL, "workspace must be 256-byte aligned");
  return RS_OK;
}

template <typename T>
rs_status pack_impl(const T* C, const T* S, int64_t ldcs, int64_t m, int64_t n, int64_t k, int side, int order,
                    int kind, void* ws, size_t bytes, void* stream) {
  Geometry g;
  const int dtype = sizeof(T) == 8 ? RS_DTYPE_F64 : RS_DTYPE_F32;
  rs_status rc = validate(m, n, m > 1 ? m : 1, ldcs, k, side, order, kind, dtype, true, &g);
  if (rc != RS_OK) return rc;
  if (!C || !S) return fail(RS_EINVAL, "null pointer");
  rc = check_workspace(g, ws, bytes);
  if (rc != RS_OK) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int rev = order == RS_ORDER_REVERSE;
  return kind == RS_KIND_REFLECTOR ? launch_pack<T, true>(g, C, S, ldcs, rev, ws, st)
                                   : launch_pack<T, false>(g, C, S, ldcs, rev, ws, st);
}

template <typename T>
rs_status apply_packed_impl(T* A, int64_t m, int64_t n, int64_t lda, int64_t k, int side, int order, int kind,
                            int strict, void* ws, size_t bytes, void* stream) {
  Geometry g;
  const int dtype = sizeof(T) == 8 ? RS_DTYPE_F64 : RS_DTYPE_F32;
  rs_status rc = validate(m, n, lda, 0, k, side, order, kind, dtype, false, &g);
  if (rc != RS_OK) return rc;
  if (g.owners == 0) return RS_OK;
  if (!A) return fail(RS_EINVAL, "null pointer");
  rc = check_workspace(g, ws, bytes);
  if (rc != RS_OK) return rc;
  return run_dispatch<T>(g, A, order == RS_ORDER_REVERSE, kind, strict, ws, reinterpret_cast<cudaStream_t>(stream));
}

template <typename T>
rs_status apply_impl(int algo, T* A, int64_t m, int64_t n, int64_t lda, const T* C, const T* S, int64_t ldcs,
                     int64_t k, int side, int order, int kind, int strict, void* workspace, size_t ws_bytes,
                     void* stream) {
  const int dtype = sizeof(T) == 8 ? RS_DTYPE_F64 : RS_DTYPE_F32;
  if (algo != RS_ALGO_PIPELINE && algo != RS_ALGO_NAIVE) return fail(RS_EINVAL, "unknown algorithm");
  Geometry g;
  rs_status vrc = validate(m, n, lda, ldcs, k, side, order, kind, dtype, true, &g);
  if (vrc != RS_OK) return vrc;
  if (g.owners == 0) return RS_OK;  // no rows: no-op (blocking.py:446-447)
  if (!A || !C || !S) return fail(RS_EINVAL, "null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int rev = order == RS_ORDER_REVERSE;
  if (algo == RS_ALGO_NAIVE) {
    if (strict) {
      return kind == RS_KIND_REFLECTOR ? launch_naive<T, true, true>(g, A, C, S, ldcs, rev, st)
                                       : launch_naive<T, true, false>(g, A, C, S, ldcs, rev, st);
    }
    return kind == RS_KIND_REFLECTOR ? launch_naive<T, false, true>(g, A, C, S, ldcs, rev, st)
                                     : launch_naive<T, false, false>(g, A, C, S, ldcs, rev, st);
  }
  const size_t need = g.coef_bytes + g.flag_bytes;
  void* ws = workspace;
  bool owned = false;
  if (ws == nullptr) {
    cudaError_t e = cudaMallocAsync(&ws, need, st);
    if (e != cudaSuccess) return fail(RS_ENOMEM, std::string("workspace allocation: ") + cudaGetErrorString(e));
    owned = true;
  } else if (ws_bytes < need) {
    return fail(RS_ENOMEM, "workspace smaller than rs_workspace_bytes()");
  } else if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) {
    return fail(RS_EINVAL, "workspace must be 256-byte aligned");
  }
  rs_status rc = kind == RS_KIND_REFLECTOR ? launch_pack<T, true>(g, C, S, ldcs, rev, ws, st)
                                           : launch_pack<T, false>(g, C, S, ldcs, rev, ws, st);
  if (rc == RS_OK) rc = run_dispatch<T>(g, A, rev, kind, strict, ws, st);
  if (owned) {
    cudaError_t e = cudaFreeAsync(ws, st);
    if (rc == RS_OK && e != cudaSuccess) return fail(RS_ECUDA, std::string("cudaFreeAsync: ") + cudaGetErrorString(e));
  }
  return rc;
}

// ------------------------------------------------------------------------------------
// FMA-pipe peak probe (roofline denominator: MEASURED_PEAKS.json has no FP64/FP32 entry)
// ------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) rs_fma_peak_kernel(T* out, int iters, T a, T b) {
  T acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma_rn(acc[c], a, b);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == (T)-1.2345) out[0] = s;
}

template <typename T>
rs_status fma_peak(double* tflops, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  T* out = nullptr;
  if (cudaMallocAsync(&out, 64, st) != cudaSuccess) return fail(RS_ENOMEM, "peak probe allocation");
  const int iters = sizeof(T) == 8 ? 20000 : 40000;
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  rs_fma_peak_kernel<T><<<blocks, threads, 0, st>>>(out, iters, (T)0.999, (T)0.001);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, st);
    rs_fma_peak_kernel<T><<<blocks, threads, 0, st>>>(out, iters, (T)0.999, (T)0.001);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, st);
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("peak probe: ") + cudaGetErrorString(e));
  *tflops = 2.0 * 8.0 * (double)iters * blocks * threads / (best * 1e-3) / 1e12;
  return RS_OK;
}

}  // namespace

extern "C" {

rs_status rs_fma_peak_tflops(int dtype, double* tflops, void* stream) {
  g_err.clear();
  if (!tflops) return fail(RS_EINVAL, "null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return dtype == RS_DTYPE_F32 ? fma_peak<float>(tflops, st) : fma_peak<double>(tflops, st);
}

int rs_version(void) { return RS_VERSION; }

const char* rs_last_error(void) { return g_err.c_str(); }

size_t rs_workspace_bytes(int64_t m, int64_t n, int64_t k, int side, int kind, int dtype) {
  if (m < 0 || n < 0 || k < 1) return 0;
  if (side != RS_SIDE_RIGHT && side != RS_SIDE_LEFT) return 0;
  if (kind != RS_KIND_ROTATION && kind != RS_KIND_REFLECTOR) return 0;
  if (dtype != RS_DTYPE_F64 && dtype != RS_DTYPE_F32) return 0;
  const int64_t len = side == RS_SIDE_LEFT ? m : n;
  if (len < 2) return 0;
  Geometry g;
  make_geometry(m, n, m > 1 ? m : 1, k, side, kind, dtype, &g);
  return g.coef_bytes + g.flag_bytes;
}

rs_status rs_apply_f64(double* A, int64_t m, int64_t n, int64_t lda, const double* C, const double* S, int64_t ldcs,
                       int64_t k, int side, int order, int kind, int strict, void* workspace, size_t workspace_bytes,
                       void* stream) {
  g_err.clear();
  return apply_impl<double>(RS_ALGO_PIPELINE, A, m, n, lda, C, S, ldcs, k, side, order, kind, strict, workspace,
                            workspace_bytes, stream);
}

rs_status rs_apply_f32(float* A, int64_t m, int64_t n, int64_t lda, const float* C, const float* S, int64_t ldcs,
                       int64_t k, int side, int order, int kind, int strict, void* workspace, size_t workspace_bytes,
                       void* stream) {
  g_err.clear();
  return apply_impl<float>(RS_ALGO_PIPELINE, A, m, n, lda, C, S, ldcs, k, side, order, kind, strict, workspace,
                           workspace_bytes, stream);
}

rs_status rs_apply_algo_f64(int algo, double* A, int64_t m, int64_t n, int64_t lda, const double* C, const double* S,
                            int64_t ldcs, int64_t k, int side, int order, int kind, int strict, void* workspace,
                            size_t workspace_bytes, void* stream) {
  g_err.clear();
  return apply_impl<double>(algo, A, m, n, lda, C, S, ldcs, k, side, order, kind, strict, workspace,
                            workspace_bytes, stream);
}

rs_status rs_apply_algo_f32(int algo, float* A, int64_t m, int64_t n, int64_t lda, const float* C, const float* S,
                            int64_t ldcs, int64_t k, int side, int order, int kind, int strict, void* workspace,
                            size_t workspace_bytes, void* stream) {
  g_err.clear();
  return apply_impl<float>(algo, A, m, n, lda, C, S, ldcs, k, side, order, kind, strict, workspace,
                           workspace_bytes, stream);
}

rs_status rs_plan_info(int64_t m, int64_t n, int64_t k, int side, int kind, int dtype, int* grid_ctas,
                       int* warps_per_cta, int64_t* units, int* band_width, int* rows_per_tile, size_t* smem_bytes) {
  g_err.clear();
  if (m < 0 || n < 0 || k < 1) return fail(RS_EINVAL, "bad dimensions");
  const int64_t len = side == RS_SIDE_LEFT ? m : n;
  if (len < 2) return fail(RS_EINVAL, "rotated dimension must be >= 2");
  Geometry g;
  make_geometry(m, n, m > 1 ? m : 1, k, side, kind, dtype, &g);
  LaunchPlan lp;
  rs_status rc = plan_launch(g, dtype == RS_DTYPE_F64 ? 8 : 4, kernel_variant(), &lp);
  if (rc != RS_OK) return rc;
  if (grid_ctas) *grid_ctas = lp.grid;
  if (warps_per_cta) *warps_per_cta = lp.nw;
  if (units) *units = lp.units;
  if (band_width) *band_width = kK;
  if (rows_per_tile) *rows_per_tile = lp.variant == VAR_V1 ? kTileOwners : (32 / lp.variant) * kR;
  if (smem_bytes) *smem_bytes = lp.smem;
  return RS_OK;
}

int64_t rs_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

rs_status rs_pack_f64(const double* C, const double* S, int64_t ldcs, int64_t m, int64_t n, int64_t k, int side,
                      int order, int kind, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  return pack_impl<double>(C, S, ldcs, m, n, k, side, order, kind, workspace, workspace_bytes, stream);
}
rs_status rs_pack_f32(const float* C, const float* S, int64_t ldcs, int64_t m, int64_t n, int64_t k, int side,
                      int order, int kind, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  return pack_impl<float>(C, S, ldcs, m, n, k, side, order, kind, workspace, workspace_bytes, stream);
}
rs_status rs_apply_packed_f64(double* A, int64_t m, int64_t n, int64_t lda, int64_t k, int side, int order, int kind,
                              int strict, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  return apply_packed_impl<double>(A, m, n, lda, k, side, order, kind, strict, workspace, workspace_bytes, stream);
}
rs_status rs_apply_packed_f32(float* A, int64_t m, int64_t n, int64_t lda, int64_t k, int side, int order, int kind,
                              int strict, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  return apply_packed_impl<float>(A, m, n, lda, k, side, order, kind, strict, workspace, workspace_bytes, stream);
}

rs_status rs_debug_set_trace(void* device_ptr) {
  g_err.clear();
#ifndef RS_TRACE
  (void)device_ptr;
  return fail(RS_EUNSUPPORTED, "library built without -DRS_TRACE");
#endif
  unsigned long long* p = reinterpret_cast<unsigned long long*>(device_ptr);
  (void)kTraceWords;
  cudaError_t e = cudaMemcpyToSymbol(g_trace, &p, sizeof(p));
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("rs_debug_set_trace: ") + cudaGetErrorString(e));
  return RS_OK;
}

}  // extern "C"
