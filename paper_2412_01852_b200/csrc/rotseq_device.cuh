// rotseq_device.cuh — device side of the B200 rotation-sequence library: records,
// arithmetic, PTX helpers, the work split, the persistent pipeline kernel and the
// pack / naive / peak kernels. Included by rotseq_b200.cu (host side + C-ABI) and by
// pipeline_variant.cu, which is compiled once per (dtype, strict, kind) so the eight
// pipeline-kernel families build in parallel. See rotseq_b200.cu for the design notes.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "rotseq_b200.h"

namespace rsk {
// ------------------------------------------------------------------------------------
// compile-time geometry
// ------------------------------------------------------------------------------------
constexpr int kK = 8;          // sweeps per unit window (lanes of the wavefront), default
// Wide windows (measured and rejected; off by default): with RS_F32_WIDE=1,
// fp32 right-side launches whose units all span >= 9 sweeps use a 16-sweep window
// (17-column blocks), with RS_F64_WIDE=1 fp64 ones a 12-sweep window. Fewer hand-offs per
// flop, but the fully unrolled block body no longer fits the instruction cache (fp32
// config 4: 33.2 -> 11.4 TF/s). The env RS_F32_K8=1 / RS_F64_K8=1 turns them off at run time.
#ifndef RS_F32_WIDE
#define RS_F32_WIDE 0
#endif
#ifndef RS_F64_WIDE
#define RS_F64_WIDE 0
#endif
__host__ __device__ constexpr int wide_k(size_t tsz) { return tsz == 4 ? 16 : 12; }
// owners (rows) per thread, per element size. 2 for both: fp32 with 4 rows per thread (8
// warps of 255 registers per CTA) measured 30.3 TF/s at config 4 against 31.1 with 2.
#ifndef RS_ROWS_F32
#define RS_ROWS_F32 2
#endif
#ifndef RS_ROWS_F64
#define RS_ROWS_F64 2
#endif
__host__ __device__ constexpr int rows_for(size_t tsz) { return tsz == 4 ? RS_ROWS_F32 : RS_ROWS_F64; }
constexpr int kRMax = 4;
#ifndef RS_FLAG_EVERY
#define RS_FLAG_EVERY 8
#endif
#ifndef RS_FLAG_TAIL
#define RS_FLAG_TAIL 1  // progress is published every block in the last RS_FLAG_TAIL blocks
#endif
#ifndef RS_STAGES
#define RS_STAGES 2
#endif
#ifndef RS_STAGES_F32
#define RS_STAGES_F32 2
#endif
// ring depth in chunks of K+1 columns (self-fill runs S-1 ahead). 3-chunk fp32 rings
// measured 2.4% slower at config 4 (the larger shared-memory carve-out shrinks L1).
__host__ __device__ constexpr int stages_for(size_t tsz) { return tsz == 4 ? RS_STAGES_F32 : RS_STAGES; }
// Right-side rings can hand chunks over in kSub sub-chunks of (K+1)/kSub columns (the
// consumer starts a block once its first columns are in): one "full" barrier per
// (slot, sub-chunk). RS_SUBCHUNK=1 enables it (default off: 1 sub-chunk).
#ifndef RS_SUBCHUNK
#define RS_SUBCHUNK 0
#endif
constexpr int kSub = RS_SUBCHUNK ? 3 : 1;
__host__ __device__ constexpr int full_bars(int stages, bool left) { return left ? stages : stages * kSub; }
// per-warp control words: full barriers, the consumed counter, two coefficient barriers
__host__ __device__ constexpr int ctl_words(int stages, bool left) { return full_bars(stages, left) + 3; }
#ifndef RS_RIGHT_LEAN
#define RS_RIGHT_LEAN 0
#endif
#ifndef RS_STS_DIRECT
#define RS_STS_DIRECT 1
#endif
#ifndef RS_FMA_PAIRED
#define RS_FMA_PAIRED 0
#endif
#ifndef RS_MAX_WARPS
#define RS_MAX_WARPS 16
#endif
constexpr int kMaxWarps = RS_MAX_WARPS;  // warps per CTA upper bound (launch bounds)
// Left side: the owner-major chunk copies need more registers; 12 warps (170 registers per
// thread) keep the unrolled body free of spills.
constexpr int kMaxWarpsLeft = 12;
// 4 rows per thread need the register budget of 8-warp CTAs (255 per thread)
// The 16-sweep window (34-register window + wider coefficient queue) gets the register
// budget of RS_WIDE_WARPS-warp CTAs.
#ifndef RS_WIDE_WARPS
#define RS_WIDE_WARPS 12
#endif
#ifndef RS_WIDE_WARPS_F64
#define RS_WIDE_WARPS_F64 8
#endif
#ifndef RS_R4_WARPS
#define RS_R4_WARPS 8
#endif
__host__ __device__ constexpr int max_warps_for(size_t tsz, bool left, int K = 8) {
  return K > 8 ? (tsz == 8 ? RS_WIDE_WARPS_F64 : RS_WIDE_WARPS)
               : (rows_for(tsz) == 4 ? RS_R4_WARPS : (left ? kMaxWarpsLeft : kMaxWarps));
}
__host__ __device__ constexpr int tile_owners(size_t tsz) { return 32 * rows_for(tsz); }
constexpr uint32_t kSuspendHintNs = 1000000;  // mbarrier try_wait suspend-time hint
constexpr int kFlagEvery = RS_FLAG_EVERY;   // hand-off progress is published every 8 blocks (fence cost)
constexpr size_t kTrashBytes = 32 * kRMax * 8;  // scratch slot per lane for rows past the matrix

enum : int { SRC_RING = 0, SRC_GLOBAL = 1, SRC_FLAG = 2 };
enum : int { DST_RING = 0, DST_GLOBAL = 1, DST_FLAG = 2 };


// ------------------------------------------------------------------------------------
// coefficient records and arithmetic
// ------------------------------------------------------------------------------------
template <typename T, bool REFL>
struct Coef;
template <>
struct alignas(16) Coef<double, false> {
  double c, s;
};
template <>
struct alignas(16) Coef<float, false> {
  // fp32 rotations travel in pairs: lanes 2i and 2i+1 of a wave share one 16-byte record
  // (c, s, c', s'), so one broadcast LDS.128 serves two rotations (see kPairRecs)
  float c, s, pad0, pad1;
};
template <typename T>
struct alignas(4 * sizeof(T)) Coef<T, true> {
  T s, d, e, pad;  // d = c - s, e = c + s (hoisted exactly as core.py:142-143)
};
// Scaled ("fast Givens") records: (tau1, -tau2), see rs_pack_scaled_kernel.
template <typename T>
using SCoef = Coef<T, false>;
// per block of a scaled-form unit: the K+1 column scales (working type) in 16-byte records
__host__ __device__ constexpr int scale_recs(int K, size_t tsz) { return (int)(((K + 1) * tsz + 15) / 16); }
// blocks per coefficient buffer: the right side copies them in pairs; the left side (whose
// global chunk copies go through L1, which shares the SRAM with shared memory) one by one
__host__ __device__ constexpr int coef_blocks_per_buf(bool left) { return left ? 1 : 2; }

// fp32 rotation records (standard and scaled) hold two lanes each; everything else one.
// A unit of width kb then stores recs_per_wave(kb) records per wave; units keep the
// record offsets of the one-lane layout (p0 * nblk * (K+1)), so the pair layout only uses
// the first part of each unit's region.
template <typename T, bool REFL>
constexpr bool kPairRecs = sizeof(T) == 4 && !REFL;
__host__ __device__ constexpr int recs_per_wave(int kb, bool pair) { return pair ? (kb + 1) / 2 : kb; }
// the (c, s) of lane l from a wave's records
template <bool PAIR, typename CoefT>
__device__ __forceinline__ CoefT lane_coef(const CoefT* __restrict__ wrec, int l) {
  if constexpr (PAIR) {
    const CoefT r = wrec[l >> 1];
    CoefT o = r;
    if (l & 1) {
      o.c = r.pad0;
      o.s = r.pad1;
    }
    return o;
  } else {
    return wrec[l];
  }
}

// bytes of one per-warp coefficient buffer (two per warp: double buffering)
// (one block of a unit of the widest width K: (K+1) waves of recs_per_wave(K) records, plus
// the scaled form's column scales; host mirror: smem_per_warp in rotseq_b200.cu)
__host__ __device__ constexpr size_t coef_block_bytes(int K, bool pair, size_t rec, size_t tsz) {
  const size_t std_bytes = (size_t)(K + 1) * (pair ? (K + 1) / 2 : K) * rec;
  const size_t scl_bytes = ((size_t)(K + 1) * (pair ? (K + 1) / 2 : K) + scale_recs(K, tsz)) * 16;
  return std_bytes > scl_bytes ? std_bytes : scl_bytes;
}
template <typename T, bool REFL, int K = kK>
__host__ __device__ constexpr size_t coef_buf_bytes() {
  return coef_block_bytes(K, kPairRecs<T, REFL>, sizeof(Coef<T, REFL>), sizeof(T));
}

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
// Scaled form (fast mode): the window holds x~ = x / sigma_x per column; one rotation is
//   x~' = x~ + tau1 * y~ ,  y~' = y~ - tau2 * x~      (2 FMAs instead of 2 MUL + 2 FMA)
template <typename T>
__device__ __forceinline__ void xform_scaled(T& x, T& y, const SCoef<T>& cf) {
  const T xo = x;
  x = fma_rn(cf.c, y, x);
  y = fma_rn(cf.s, xo, y);
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
// The suspend-time hint parks a waiting warp in hardware until the phase completes instead
// of spinning: spinning waits would steal issue slots from the warps sharing its SM
// sub-partition (measured: ~14% of all issued instructions without the hint).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// RS_WAIT_MODE (measurement knob): 0 try_wait with a suspend-time hint (default), 1
// try_wait without a hint, 2 test_wait + nanosleep back-off
#ifndef RS_WAIT_MODE
#define RS_WAIT_MODE 0
#endif
#ifndef RS_WAIT_NS
#define RS_WAIT_NS 64
#endif
__device__ __forceinline__ void mbar_wait_addr(uint32_t bar, uint32_t parity) {
#if RS_WAIT_MODE == 1
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "RS_WAITN_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra RS_WAITN_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
#elif RS_WAIT_MODE == 2
  uint32_t ok;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) break;
    __nanosleep(RS_WAIT_NS);
  }
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "RS_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra RS_WAIT_%=;\n}" ::"r"(bar),
      "r"(parity), "r"(kSuspendHintNs)
      : "memory");
#endif
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_test(bar, parity)) return;  // already complete: skip try_wait's fixed latency
  mbar_wait_addr(smem_u32(bar), parity);
}
// Address-based forms (shared-window u32 addresses computed once per warp) and single-lane
// forms predicated inside the asm, so the per-block protocol has no divergent branches.
__device__ __forceinline__ bool mbar_test_a(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  if (mbar_test_a(bar, parity)) return;
  mbar_wait_addr(bar, parity);
}
__device__ __forceinline__ void mbar_arrive_if(uint32_t bar, bool pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
      "@p mbarrier.arrive.shared::cta.b64 _, [%0];\n}" ::"r"(bar),
      "r"((uint32_t)pred)
      : "memory");
}
// "consumed" counters: relaxed stores. Every ring read of the released chunk has already
// returned its data (the values were consumed by the block's FMAs or stores before the
// warp barrier), so no later write to the slot can be observed by those reads.
__device__ __forceinline__ void st_shared_u32_if(uint32_t a, uint32_t v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
      "@p st.volatile.shared::cta.u32 [%0], %1;\n}" ::"r"(a),
      "r"(v), "r"((uint32_t)pred)
      : "memory");
}
// coefficient block copy by one lane: arm the barrier with the byte count, start the copy
__device__ __forceinline__ void coef_copy_if(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, bool pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %4, 0;\n\t"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t"
      "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "r"((uint32_t)pred)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// TMA bulk copy global -> shared completing `bytes` of transaction count on `bar`.
__device__ __forceinline__ void bulk_g2s_nowait(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
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
#ifndef RS_CSLEEP
#define RS_CSLEEP 32
#endif
  while (ld_acquire_shared(p) < target) __nanosleep(RS_CSLEEP);
}
__device__ __forceinline__ uint32_t wait_flag(const uint32_t* p, uint32_t target) {
  uint32_t v;
  while ((v = ld_acquire(p)) < target) __nanosleep(64);
  return v;
}

// Debug-only instrumentation (compiled in with -DRS_TRACE; see rs_debug_set_trace).
// Each unit a warp runs writes one record of kTraceWords uint64 to
// trace[((cta * kMaxWarps + warp) * kTraceRounds + round) * kTraceWords]:
//   0 tile | src<<40 | dst<<44 | smid<<48, 1 globaltimer at unit start, 2 at unit end,
//   3 cycles issuing self-fill / waiting for progress flags, 4 coefficient waits, 5 ring-full
//   waits, 6 ring-space waits, 7 compute (run_block), 8 post-block hand-off work, 9 p0 | kb<<32.
constexpr int kTraceWords = 10;
constexpr int kTraceRounds = 32;
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
__device__ __forceinline__ void trace_unit(unsigned long long* t, int warp, int jr, long long tile, int p0, int kb,
                                           int src, int dst, const TraceAcc& acc) {
#ifdef RS_TRACE
  if (t != nullptr && (threadIdx.x & 31) == 0 && jr < kTraceRounds) {
    unsigned long long* rec = t + (((size_t)blockIdx.x * kMaxWarps + warp) * kTraceRounds + jr) * kTraceWords;
    rec[0] = (unsigned long long)tile | ((unsigned long long)src << 40) | ((unsigned long long)dst << 44) |
             ((unsigned long long)trace_smid() << 48);
    rec[1] = acc.t0;
    rec[2] = trace_gtime();
    for (int i = 0; i < 6; ++i) rec[3 + i] = acc.c[i];
    rec[9] = (unsigned long long)p0 | ((unsigned long long)kb << 32);
  }
#else
  (void)t, (void)warp, (void)jr, (void)tile, (void)p0, (void)kb, (void)src, (void)dst, (void)acc;
#endif
}

// ------------------------------------------------------------------------------------
// kernel parameters
// ------------------------------------------------------------------------------------
struct PipeParams {
  void* A;           // element (owner o, wave-column v) at A + o*os + v*cs
  long long os;      // owner stride (elements)
  long long cs;      // wave-column stride (elements, negative for reverse order)
  long long owners;  // independent lines (rows for right side, columns for left)
  long long tiles;   // ceil(owners / 64)
  long long units;   // U: (tile, sweep-range) units in total
  long long t1;      // the first t1 tiles hold ua+1 units, the others ua
  const void* coef;  // packed coefficient blocks (see rs_pack_kernel)
  const void* coef_scaled;  // scaled-form blocks (rs_pack_scaled_kernel)
  const uint32_t* unsafe;   // [2][ua+1] per (sweep partition, unit index): set by rs_pack_scaled_kernel
                            // when the unit's coefficients are outside the scaled form's safe range
  uint32_t* flags;   // [tiles*k + 1] progress flags of in-place hand-offs, index tile*k + p0
  void* trash;       // 32*R elements: write/read target of lanes past the last row
  int ua;            // units per tile (base)
  int len;           // length of the rotated dimension (n right, m left)
  int k;             // sweeps
  int nchunk;        // ceil(len / (K+1))
  int nblk;          // nchunk + 1
  int nw;            // warps per CTA (multiple of 4)
  int use_scaled;    // fast fp64: scaled records were packed
  int credit;        // ring credit in chunks (1..S)
  int ring_sts;      // right side: ring outputs through STS (else the generic store path)
  // host-streaming mode (rs_apply_host_*): A arrives from the host in wave-column chunks
  // of cw columns while the kernel runs, and leaves in the same chunks as soon as every
  // tile's final unit has emitted them. Null pointers: A is resident.
  const uint32_t* arrived;  // number of chunks already copied in (written by the copy stream)
  uint32_t* done;           // per chunk: tiles whose final unit has emitted it
  int cw;                   // chunk width in wave columns
  int ncw;                  // number of chunks
  unsigned long long* trace;  // debug timeline buffer (RS_TRACE builds), or null
  int sweep_off;     // offset of the sweep split (sweep_start), 0 <= sweep_off < units per tile
};

// ------------------------------------------------------------------------------------
// work split. The U units are numbered tile-major; tile t holds u_t = ua (+1 for t < t1)
// units whose sweep ranges split the k sweeps evenly: unit i of the tile covers sweeps
// [floor(i*k/u_t), floor((i+1)*k/u_t)) (width <= K). The planner picks U = 4*G*q so every
// CTA runs 4q consecutive units and, with position p on warp p % NW (NW a multiple of 4),
// every SM sub-partition runs q units of nearly equal total width.
// ------------------------------------------------------------------------------------
struct Unit {
  long long tile;
  int p0;  // first sweep
  int kb;  // sweeps (1..kK)
};
// First sweep of unit i (of ut) of a tile: the k sweeps split evenly. (Uneven splits —
// a narrower head unit, widths tapered along the chain — measured much slower: a chain
// runs at the pace of its widest unit.)
// `off` (0 <= off < ut) shifts where the wider units of an uneven split fall inside a chain
// (the ends stay 0 and k): with off = 0 the wider unit of each period comes last, which
// puts one on the chain's tail and, for some tiles, on the units that also carry a
// flag hand-off; the equal-chain plans (plan_launch) use off = ut/2.
__host__ __device__ __forceinline__ int sweep_start(long long i, int ut, int k, int off = 0) {
  if (i <= 0) return 0;
  if (i >= ut) return k;
  return (int)((i * k + off) / ut);
}
__host__ __device__ __forceinline__ long long tile_first_unit(long long t, long long t1, int ua) {
  return t < t1 ? t * (ua + 1) : t1 * (ua + 1) + (t - t1) * ua;
}
__host__ __device__ __forceinline__ Unit unit_at(long long g, long long t1, int ua, int k, int off = 0) {
  Unit u;
  const long long big = t1 * (ua + 1);
  long long i;
  int ut;
  if (g < big) {
    u.tile = g / (ua + 1);
    i = g - u.tile * (ua + 1);
    ut = ua + 1;
  } else {
    const long long r = g - big;
    u.tile = t1 + r / ua;
    i = r - (u.tile - t1) * ua;
    ut = ua;
  }
  u.p0 = sweep_start(i, ut, k, off);
  u.kb = sweep_start(i + 1, ut, k, off) - u.p0;
  return u;
}
// CTA c runs units [g0, g1). When the range ends inside a tile whose first unit lies inside
// the range, that last partial tile (it feeds the next CTA) runs first: nl > 0 units.
struct CtaRange {
  long long g0, g1;
  int nl;
};
__host__ __device__ __forceinline__ CtaRange cta_range(long long U, long long c, long long G, long long t1, int ua,
                                                       int k, int off = 0) {
  CtaRange r;
  r.g0 = U * c / G;
  r.g1 = U * (c + 1) / G;
  r.nl = 0;
  if (r.g1 > r.g0) {
    const Unit last = unit_at(r.g1 - 1, t1, ua, k, off);
    if (last.p0 + last.kb < k) {
      const long long f = tile_first_unit(last.tile, t1, ua);
      if (f > r.g0) r.nl = (int)(r.g1 - f);
    }
  }
  return r;
}
__host__ __device__ __forceinline__ long long pos_to_unit(const CtaRange& r, long long p) {
  return p < r.nl ? r.g1 - r.nl + p : r.g0 + p - r.nl;
}
__host__ __device__ __forceinline__ long long unit_to_pos(const CtaRange& r, long long g) {
  return g >= r.g1 - r.nl ? g - (r.g1 - r.nl) : g - r.g0 + r.nl;
}

// Unit widths a window of K sweeps is compiled for: every width 1..8 for the 8-sweep
// window; the 16-sweep window (fp32, right side) only runs units of 9..16 sweeps (the
// planner guarantees it; narrower units use the 8-sweep window).
__host__ __device__ constexpr int kb_min(int K) { return K > 8 ? 9 : 1; }
template <int K, int KMIN, int KB = K, typename F>
__device__ __forceinline__ void dispatch_width(int Kb, F&& f) {
  if constexpr (KB >= KMIN) {
    if (Kb == KB || KB == KMIN) {
      f(std::integral_constant<int, KB>{});
    } else {
      dispatch_width<K, KMIN, KB - 1>(Kb, f);
    }
  }
}

// ------------------------------------------------------------------------------------
// one block of K+1 waves for one warp (fully unrolled; window slots are compile-time)
//   block b covers waves t = b(K+1)-1 .. b(K+1)+K-1. At the start of wave u it emits
//   column (b-1)(K+1)+u (finished after wave t-1) through the output pointers, then loads
//   column b(K+1)+u into slot u; lane l < KB rotates columns (t-l, t-l+1) = slots
//   (u-1-l, u-l) with record cb[u*KB+l]. Output goes to the next unit's ring (shared)
//   or to A (global) through one generic store path, so a unit width compiles to ONE loop
//   body (instruction-cache footprint). EDGE blocks check every column and lane at run time.
// ------------------------------------------------------------------------------------
// OUTS: the output columns go to shared memory (the next unit's ring, or the left side's
// staging slot) at obase + u*OSU + r*OSR elements and are stored with STS; otherwise to A
// through the generic pointers op[r] (stride ostr[r]).
// FIRST (with EDGE): block 0 of a unit whose first chunk lies inside the matrix (the caller
// guarantees len >= K+1): nothing to emit, every column of the chunk valid, and rotation
// (u, l) in range iff l < u — a compile-time triangle, so half of the block's rotations
// vanish and the rest carry one width test instead of the generic edge tests.
// final_exit (EDGE, the draining last block): the unit's work ends with the store of column
// len-1; when `early_out` is set (ring output) the consumer's "full" barrier is signalled
// right there, and the rest of the block (rotations that are all out of range) is skipped.
// Both shorten the hand-off lag per chain hop.
// CDQ: depth of the register queue of prefetched coefficient records. 4 everywhere except the
// 168-register fp64 right-side build, where 6 measures +2.3% (config 2: 19.4 -> 19.9 TF/s per
// step; 2 / 3 / 8: 19.7 / 19.5 / 19.7) — and -2.5% on the 128-register build (config 3).
#ifndef RS_COEF_QUEUE
#define RS_COEF_QUEUE 4
#endif
#ifndef RS_COEF_QUEUE_SMALL
#define RS_COEF_QUEUE_SMALL 6
#endif
template <typename T, int K, int R, int KB, bool STRICT, bool REFL, bool EDGE, bool SCALED, bool LEFT, bool OUTS,
          bool FIRST = false, int CDQ = RS_COEF_QUEUE>
__device__ __forceinline__ void run_block(T (&w)[R][K + 1],
                                          const std::conditional_t<SCALED, SCoef<T>, Coef<T, REFL>>* __restrict__ cb,
                                          const T* islot, T* const (&op)[R], const long long (&ostr)[R],
                                          T* obase, int b, int len, int Kb, int lane, bool has_in_rt,
                                          bool has_out_rt, uint64_t* sub_in = nullptr, uint32_t sub_par = 0,
                                          uint64_t* sub_out = nullptr, bool final_exit = false,
                                          uint64_t* early_out = nullptr) {
  static_assert(!FIRST || EDGE, "FIRST is a variant of the edge block");
  // sub-chunk hand-off (kSub > 1, right side): wait for sub-chunk h before loading its first
  // column; announce sub-chunk h once its last column is stored
  constexpr int SUBW = (K + 1) / kSub;
  // OUTS: element strides of the output column (u) and row (r) in the shared slot
  constexpr int OSU = LEFT ? 1 : 32 * R;
  constexpr int OSR = LEFT ? 32 * (K + 1) : 32;
  constexpr int TR = 32 * R;
  constexpr int NL = EDGE ? K : KB;
  // edge-block index arithmetic: 32-bit on the fp64 right side (columns fit an int: len is
  // one; +1.3% at configs 2 and 3), 64-bit elsewhere (the left-side and fp32 bodies
  // schedule better with it: -4% / -1% at configs 5 / 4 otherwise)
  using IdxT = std::conditional_t<(!LEFT && sizeof(T) == 8), int, long long>;
  const IdxT c0 = (IdxT)b * (K + 1);
  const bool has_in = !EDGE || FIRST || has_in_rt;
  const bool has_out = !FIRST && (!EDGE || has_out_rt);
  // scaled mode: the emitted column is multiplied back by its scale (after the block's records)
  constexpr bool PAIR = kPairRecs<T, REFL>;
  const int NR = recs_per_wave(EDGE ? Kb : KB, PAIR);  // records per wave
  const T* __restrict__ sc = reinterpret_cast<const T*>(cb + (K + 1) * NR);
  T* q[R];
#pragma unroll
  for (int r = 0; r < R; ++r) q[r] = op[r];
  auto load_col = [&](int u, T (&dst)[R]) {
    const IdxT col = c0 + u;
    if (!EDGE || FIRST || (has_in && col < len)) {
#pragma unroll
      for (int r = 0; r < R; ++r) dst[r] = islot[LEFT ? (lane + 32 * r) * (K + 1) + u : u * TR + lane + 32 * r];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) dst[r] = T(0);
    }
  };
  T nxt[R];
  load_col(0, nxt);
  // coefficient records prefetched CD rotation steps ahead (register queue; the ring index
  // t % CD is a compile-time constant in the unrolled loops)
  using CoefT = std::conditional_t<SCALED, SCoef<T>, Coef<T, REFL>>;
  constexpr int CD = CDQ;
  CoefT cq[CD];
  if constexpr (!EDGE) {
#pragma unroll
    for (int t = 0; t < CD && t < (K + 1) * NL; ++t) cq[t] = lane_coef<PAIR>(cb + (t / NL) * NR, t % NL);
  }
#pragma unroll
  for (int u = 0; u <= K; ++u) {
    // incoming column (LEFT rings are owner-major [owner][K+1]; right rings wave-major),
    // loaded one wave ahead so the shared-memory latency overlaps the previous wave
    T nv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) nv[r] = nxt[r];
    if constexpr (kSub > 1) {
      if (u < K && (u + 1) % SUBW == 0 && sub_in != nullptr) mbar_wait(&sub_in[(u + 1) / SUBW], sub_par);
    }
    if (u < K) load_col(u + 1, nxt);
    // outgoing column (LEFT may stage it in place of the column just read)
    if (has_out) {
      const IdxT col = c0 - (K + 1) + u;
      if (!EDGE || col < len) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const T v = SCALED ? mul_rn(w[r][u], sc[u]) : w[r][u];
          if constexpr (OUTS) {
            obase[u * OSU + r * OSR] = v;
          } else {
            *q[r] = v;
          }
        }
      }
      if constexpr (!OUTS) {
#pragma unroll
        for (int r = 0; r < R; ++r) q[r] += ostr[r];
      }
      if constexpr (kSub > 1) {
        if (u % SUBW == SUBW - 1 && sub_out != nullptr) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&sub_out[u / SUBW]);
        }
      }
      if constexpr (EDGE && !FIRST) {
        if (final_exit && col == (IdxT)len - 1) {  // the unit's last column is out
          if (early_out != nullptr) {
            __syncwarp();
            if (lane == 0) mbar_arrive(early_out);
          }
          return;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) w[r][u] = nv[r];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      constexpr int M = K + 1;
      const int sx = (u - 1 - l + 2 * M) % M;
      const int sy = (sx + 1) % M;
      if constexpr (FIRST) {
        if (l >= u) continue;  // j = u - 1 - l < 0 (compile time)
        if (l >= Kb) continue;
      } else if (EDGE) {
        const IdxT j = c0 + u - 1 - l;
        if (l >= Kb || j < 0 || j > (IdxT)len - 2) continue;
      }
      // interior blocks: the record of step t = u*NL + l was loaded CD steps earlier
      CoefT cf;
      if constexpr (EDGE) {
        cf = lane_coef<PAIR>(cb + u * NR, l);
      } else {
        constexpr int NSTEP = (K + 1) * NL;
        const int t = u * NL + l;
        cf = cq[t % CD];
        if (t + CD < NSTEP) cq[t % CD] = lane_coef<PAIR>(cb + ((t + CD) / NL) * NR, (t + CD) % NL);
      }
      if constexpr (SCALED && RS_FMA_PAIRED) {
        // the R rows' FMAs with the same multiplier back to back (tau1 for every row, then
        // tau2): the shared coefficient register can come from the operand reuse cache
        T xo[R];
#pragma unroll
        for (int r = 0; r < R; ++r) xo[r] = w[r][sx];
#pragma unroll
        for (int r = 0; r < R; ++r) w[r][sx] = fma_rn(cf.c, w[r][sy], xo[r]);
#pragma unroll
        for (int r = 0; r < R; ++r) w[r][sy] = fma_rn(cf.s, xo[r], w[r][sy]);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if constexpr (SCALED) {
            xform_scaled<T>(w[r][sx], w[r][sy], cf);
          } else {
            xform<T, STRICT, REFL>(w[r][sx], w[r][sy], cf);
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// the persistent pipeline kernel
// ------------------------------------------------------------------------------------
template <typename T, int K, int R, bool STRICT, bool REFL, bool SCALED_ANY, bool HS, bool LEFT>
__device__ __forceinline__ void pipeline_units(const PipeParams& P, unsigned char* smem_raw) {
  constexpr int TR = 32 * R;
  constexpr int CHUNK = (K + 1) * TR;  // ring chunk: K+1 columns x TR owners
  constexpr size_t CBUF = coef_buf_bytes<T, REFL, K>();  // one coefficient buffer (bytes)
  constexpr int S = stages_for(sizeof(T));
  constexpr int FA = S - 1;  // self-fill distance in chunks
  static_assert(FA == 1 || FA == 2, "ring depth must be 2 or 3 chunks");
  constexpr int NBAR = ctl_words(S, LEFT);

  const int NW = P.nw;
  // warp-uniform for the compiler (uniform registers for the per-block protocol operands)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const bool lane0 = lane == 0;
  T* ring_sm = reinterpret_cast<T*>(smem_raw + (size_t)NW * 2 * coef_blocks_per_buf(LEFT) * CBUF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring_sm + (size_t)NW * S * CHUNK);

  T* const A = reinterpret_cast<T*>(P.A);
  const int len = P.len;
  const int k = P.k;
  const int nchunk = P.nchunk;
  const int nblk = P.nblk;
  const uint32_t credit = (uint32_t)P.credit;
  uint64_t* const bar_in = bars + warp * NBAR;  // in-ring of this warp: full[S], consumed, coef[2]
  uint64_t* const full_in = bar_in;
  uint32_t* const consumed_in = reinterpret_cast<uint32_t*>(bar_in + S);
  uint64_t* const cbar = bar_in + S + 1;
  // position p of a round runs on warp p % NW; the next position on warp + 1
  const int slot = warp;
  uint64_t* const full_out = bars + (warp + 1) * NBAR;
  const uint32_t* const consumed_out = reinterpret_cast<const uint32_t*>(full_out + S);
  T* const rin = ring_sm + (size_t)warp * S * CHUNK;
  T* const rout = ring_sm + (size_t)(warp + 1) * S * CHUNK;
  unsigned char* const cbuf = smem_raw + (size_t)warp * 2 * coef_blocks_per_buf(LEFT) * CBUF;
  // shared-window addresses of this warp's protocol words and buffers
  const uint32_t fullin_a = smem_u32(full_in), fullout_a = smem_u32(full_out);
  const uint32_t consin_a = smem_u32(consumed_in), cbar_a = smem_u32(cbar), cbuf_a = smem_u32(cbuf);

  const CtaRange cr = cta_range(P.units, blockIdx.x, gridDim.x, P.t1, P.ua, k, P.sweep_off);
  const long long npos = cr.g1 - cr.g0;
  uint32_t cseq = 0;  // coefficient blocks consumed by this warp (buffer = cseq&1)

  for (int jr = 0;; ++jr) {
    const long long pos = (long long)jr * NW + slot;
    if (pos >= npos) break;
    const long long g = pos_to_unit(cr, pos);
    const Unit un = unit_at(g, P.t1, P.ua, k, P.sweep_off);
    const long long tile = un.tile;
    const int p0 = un.p0;
    const int Kb = un.kb;
    // the producer of this unit is unit g-1 (same tile, ends at sweep p0); its consumer is
    // g+1. Ring hand-off when that unit is the neighbouring position of the same round.
    int src = SRC_GLOBAL, dst = DST_GLOBAL;
    if (p0 > 0) {
      src = SRC_FLAG;
      if (slot > 0 && g - 1 >= cr.g0 && unit_to_pos(cr, g - 1) == pos - 1) src = SRC_RING;
    }
    if (p0 + Kb < k) {
      dst = DST_FLAG;
      if (slot < NW - 1 && g + 1 < cr.g1 && unit_to_pos(cr, g + 1) == pos + 1) dst = DST_RING;
    }
    const bool self = src != SRC_RING;
    // arithmetic form of this unit: the scaled (fast Givens) records unless the pack
    // flagged this unit's coefficients as outside the scaled form's safe range
    const int part = tile < P.t1 ? 1 : 0;
    const long long iu = g - tile_first_unit(tile, P.t1, P.ua);
    auto unit_body = [&](auto scaled_c) {
    constexpr bool SCALED = decltype(scaled_c)::value;
    using CoefT = std::conditional_t<SCALED, SCoef<T>, Coef<T, REFL>>;

    T* grow[R];        // element (row r, column 0) of this lane's lines
    long long gcs[R];  // column stride; 0 for rows past the matrix (they use the trash slot)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long o = tile * TR + lane + 32 * r;
      const bool ok = o < P.owners;
      grow[r] = ok ? A + o * P.os : reinterpret_cast<T*>(P.trash) + lane + 32 * r;
      gcs[r] = ok ? P.cs : 0;
    }
    // LEFT coalesced chunk copies: this lane's first element e = lane is owner lo0, column
    // lv0; each step of 32 elements advances 3 owners + 5 columns (wrapping past K+1)
    static_assert(!LEFT || 32 == 3 * (K + 1) + 5, "coalesced owner-major copy assumes K + 1 = 9");
    const int lo0 = lane / (K + 1), lv0 = lane - lo0 * (K + 1);
    const long long lstep = 3 * P.os + (32 - 3 * (K + 1)) * P.cs;
    const long long lwrap = P.os - (K + 1) * P.cs;
    const T* const lbase = A + (tile * TR + lo0) * P.os + lv0 * P.cs;
    const bool lfull = tile * TR + TR <= P.owners;
    // this unit's coefficient blocks, contiguous per block (rs_pack_kernel: Kb*(K+1)
    // records; rs_pack_scaled_kernel: Kb*(K+1) records + SR records of scales)
    constexpr int SR = scale_recs(K, sizeof(T));
    const int brec = recs_per_wave(Kb, kPairRecs<T, REFL>) * (K + 1) + (SCALED ? SR : 0);
    const CoefT* ubase;
    if constexpr (SCALED) {
      ubase = reinterpret_cast<const CoefT*>(P.coef_scaled) + (size_t)part * k * nblk * (K + 1 + SR) +
              (size_t)p0 * nblk * (K + 1) + (size_t)iu * nblk * SR;
    } else {
      ubase = reinterpret_cast<const CoefT*>(P.coef) + (size_t)part * k * nblk * (K + 1) + (size_t)p0 * nblk * (K + 1);
    }
    const uint32_t blk_bytes = (uint32_t)(brec * sizeof(CoefT));
    // one elected lane: WAR fence for the buffer's previous readers, arm, start the copy
    // The buffer's previous readers are this warp's own LDS, whose values were consumed
    // before the warp barrier that precedes every issue (no proxy fence needed for WAR).
    auto issue_coef = [&](int b, uint32_t buf) {
      coef_copy_if(cbuf_a + buf * (uint32_t)(coef_blocks_per_buf(LEFT) * CBUF), ubase + (size_t)b * brec, blk_bytes, cbar_a + buf * 8u,
                   lane0);
    };
    const uint32_t seq0 = (uint32_t)jr * (uint32_t)nchunk;
    const uint32_t* myflag = P.flags + tile * k + p0;
    uint32_t* const outflag = P.flags + tile * k + p0 + Kb;
    TraceAcc tacc;
    tacc.t0 = trace_gtime();

    issue_coef(0, cseq & 1);

    // self-filled input (sweep 0 reads A; a flag hand-off reads A after the producer's
    // progress flag): cp.async (LDGSTS) straight into this warp's own ring, FA chunks ahead.
    uint32_t flag_seen = 0;
    auto fill_chunk = [&](int q) {
#ifdef RS_X_NOFILL
      if (src == SRC_GLOBAL) { cp_async_commit(); return; }
#endif
      if (src == SRC_FLAG && flag_seen < (uint32_t)q + 1) flag_seen = wait_flag(myflag, (uint32_t)q + 1);
      if (HS && src == SRC_GLOBAL) {  // host streaming: wait for the copy of these columns
        long long cend = (long long)q * (K + 1) + K;
        if (cend > len - 1) cend = len - 1;
        const uint32_t need = (uint32_t)(cend / P.cw) + 1u;
        if (flag_seen < need) flag_seen = wait_flag(P.arrived, need);
      }
      T* dstp = rin + ((seq0 + (uint32_t)q) % S) * CHUNK;
      const long long c0 = (long long)q * (K + 1);
      if constexpr (LEFT) {
        // owner-major chunk [TR owners][K+1 columns]: element e = i*32 + lane is owner
        // e/(K+1), column e%(K+1) — consecutive lanes read consecutive columns of one owner
        // (contiguous in A on the left side) and write consecutive shared words. (owner,
        // column) and the address advance incrementally (e += 32: +3 owners, +5 columns).
        int v = lv0;
        const T* sp = lbase + c0 * P.cs;
        if (lfull && c0 + K < len) {
#pragma unroll
          for (int i = 0; i < R * (K + 1); ++i) {
            cp_async_elem(dstp + i * 32 + lane, sp, true);
            v += 32 - 3 * (K + 1);
            sp += lstep;
            if (v >= K + 1) v -= K + 1, sp += lwrap;
          }
        } else {
          int ol = lo0;
#pragma unroll
          for (int i = 0; i < R * (K + 1); ++i) {
            const bool ok = tile * TR + ol < P.owners && c0 + v < len;
            cp_async_elem(dstp + i * 32 + lane, ok ? sp : A, ok);
            v += 32 - 3 * (K + 1);
            ol += 3;
            sp += lstep;
            if (v >= K + 1) v -= K + 1, ++ol, sp += lwrap;
          }
        }
        cp_async_commit();
        return;
      }
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
    unsigned long long tc = trace_clock();
    if (self) {
      fill_chunk(0);
      if (FA >= 2 && 1 < nchunk) fill_chunk(1);
      if (FA >= 2 && 1 < nchunk)
        cp_async_wait_group<1>();
      else
        cp_async_wait_group<0>();
      __syncwarp();
      mbar_arrive_if(fullin_a + (seq0 % S) * 8u, lane0);
    }
    tacc.c[0] += trace_clock() - tc;

    T w[R][K + 1];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int s = 0; s <= K; ++s) w[r][s] = T(0);

    const bool outring = dst == DST_RING;
    int done_sig = 0;  // host streaming: chunks already released by this (final) unit
    // incremental protocol state: in-ring slot / phase of the chunk read by block b
    // (iseq = seq0 + b), coefficient buffer / phase (cseq)
    uint32_t ib = seq0 % S, iph = (seq0 / S) & 1u;
    uint32_t cbi = cseq & 1u, cph = (cseq >> 1) & 1u;
    // One block: protocol + compute. KB / EDGE are compile-time so the interior loop
    // carries no per-block branches beyond this unit's hand-off protocol.
    auto block = [&](int b, auto kb_c, auto edge_c) {
      constexpr int KB = decltype(kb_c)::value;
      constexpr bool EDGE = decltype(edge_c)::value;
      unsigned long long t0 = trace_clock();
#ifdef RS_X_NOCOEF
      if (b + 1 < nblk && b < 1) issue_coef(b + 1, cbi ^ 1u);
#else
      if (b + 1 < nblk) issue_coef(b + 1, cbi ^ 1u);
#endif
      const bool has_in = !EDGE || b < nchunk;
      const bool has_out = !EDGE || b >= 1;
      if (self && b + FA < nchunk) fill_chunk(b + FA);
      unsigned long long t1 = trace_clock();
      const uint32_t iseq = seq0 + (uint32_t)b;
      const uint32_t ob = ib == 0 ? (uint32_t)(S - 1) : ib - 1u;  // slot of chunk oseq = iseq - 1
      const T* islot = rin + ib * CHUNK;
      const uint32_t oseq = iseq - 1u;
      // output: the consumer's ring slot or (LEFT) the staging slot, by shared address;
      // right side to A through generic pointers (column stride gcs)
      T* op[R];
      long long ostr[R];
      // LEFT, output to A: stage the outgoing chunk in the input slot just read (the last
      // block, which has no input, reuses the previous block's slot) and copy it out below
      const uint32_t stage_i = b < nchunk ? ib : ob;
      T* stage = rin + stage_i * CHUNK;
      // (pointers derived from the shared-memory window: plain STS with alias analysis)
      T* obase = nullptr;
      if (outring) {
        obase = rout + ob * CHUNK + lane * (LEFT ? K + 1 : 1);
      } else if (LEFT) {
        obase = rin + stage_i * CHUNK + lane * (K + 1);
      } else {
        const long long cb0 = (long long)b * (K + 1) - (K + 1);
#pragma unroll
        for (int r = 0; r < R; ++r) op[r] = grow[r] + cb0 * gcs[r], ostr[r] = gcs[r];
      }
#ifdef RS_X_NOCOEF
      if (b < 2) mbar_wait_a(cbar_a + cbi * 8u, cph);
#else
      mbar_wait_a(cbar_a + cbi * 8u, cph);
#endif
      unsigned long long t2 = trace_clock();
#ifndef RS_X_NOSYNC
      if (!self && has_in) mbar_wait_a(fullin_a + ib * 8u, iph);
#endif
      unsigned long long t3 = trace_clock();
      // ring credit: the producer runs at most `credit` chunks ahead of its consumer
#ifndef RS_X_NOSYNC
      if (outring && has_out && oseq >= credit) wait_count(consumed_out, oseq - credit + 1u);
#endif
      unsigned long long t4 = trace_clock();
      {
        const CoefT* cbp = reinterpret_cast<const CoefT*>(cbuf + cbi * coef_blocks_per_buf(LEFT) * CBUF);
        if (LEFT || outring) {
          run_block<T, K, R, KB, STRICT, REFL, EDGE, SCALED, LEFT, true>(w, cbp, islot, op, ostr, obase, b, len, Kb,
                                                                          lane, b < nchunk, b >= 1);
        } else {
          run_block<T, K, R, KB, STRICT, REFL, EDGE, SCALED, LEFT, false>(w, cbp, islot, op, ostr, nullptr, b, len, Kb,
                                                                           lane, b < nchunk, b >= 1);
        }
      }
      __syncwarp();
      if (LEFT && !outring && has_out) {  // copy the staged chunk to A, columns contiguous
        const long long cb0 = (long long)(b - 1) * (K + 1);
        int v = lv0;
        T* dp = const_cast<T*>(lbase) + cb0 * P.cs;
        if (lfull && cb0 + K < len) {
#pragma unroll
          for (int i = 0; i < R * (K + 1); ++i) {
            *dp = stage[i * 32 + lane];
            v += 32 - 3 * (K + 1);
            dp += lstep;
            if (v >= K + 1) v -= K + 1, dp += lwrap;
          }
        } else {
          int ol = lo0;
#pragma unroll
          for (int i = 0; i < R * (K + 1); ++i) {
            if (tile * TR + ol < P.owners && cb0 + v < len) *dp = stage[i * 32 + lane];
            v += 32 - 3 * (K + 1);
            ol += 3;
            dp += lstep;
            if (v >= K + 1) v -= K + 1, ++ol, dp += lwrap;
          }
        }
        __syncwarp();
      }
      unsigned long long t5 = trace_clock();
      // LEFT global output: the last block stages in the slot of chunk nchunk-1, so that
      // slot is released one block later (as nchunk, i.e. iseq of the last block)
      if (LEFT && !outring) {
        if (has_in && b + 1 < nchunk) st_shared_u32_if(consin_a, iseq + 1u, lane0);
        if (b == nchunk) st_shared_u32_if(consin_a, iseq, lane0);
      } else if (has_in) {
        st_shared_u32_if(consin_a, iseq + 1u, lane0);
      }
      if (outring && has_out) mbar_arrive_if(fullout_a + ob * 8u, lane0);
      if (dst == DST_FLAG && has_out &&
          (b < 2 * kFlagEvery || (b & (kFlagEvery - 1)) == 0 || b >= nblk - RS_FLAG_TAIL)) {
        if (lane0) {
          // the warp barrier above orders every lane's stores before lane 0's gpu-scope
          // fence; the release store then publishes "chunks 0..b-1 are in A"
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          st_release(outflag, (uint32_t)b);
        }
      }
      if (HS && dst == DST_GLOBAL && has_out && lane0) {  // host streaming: release finished chunks
        long long e = (long long)b * (K + 1) - 1;  // last column emitted by this block
        if (e > len - 1) e = len - 1;
        const int nd = e == len - 1 ? P.ncw : (int)((e + 1) / P.cw);
        if (nd > done_sig) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          for (; done_sig < nd; ++done_sig) atomicAdd(P.done + done_sig, 1u);
        }
      }
      // advance the in-ring slot (the next block reads chunk iseq + 1)
      const uint32_t nib = ib + 1u == (uint32_t)S ? 0u : ib + 1u;
      if (self && b + 1 < nchunk) {  // the chunk read by the next block has landed
        if (FA >= 2 && b + 2 < nchunk)
          cp_async_wait_group<1>();
        else
          cp_async_wait_group<0>();
        __syncwarp();
        mbar_arrive_if(fullin_a + nib * 8u, lane0);
      }
      if (nib == 0) iph ^= 1u;
      ib = nib;
#ifdef RS_X_NOCOEF
      if (b < 2) { ++cseq; cbi ^= 1u; if (cbi == 0) cph ^= 1u; }
#else
      ++cseq;
      cbi ^= 1u;
      if (cbi == 0) cph ^= 1u;
#endif
      unsigned long long t6 = trace_clock();
      tacc.c[0] += t1 - t0;
      tacc.c[1] += t2 - t1;
      tacc.c[2] += t3 - t2;
      tacc.c[3] += t4 - t3;
      tacc.c[4] += t5 - t4;
      tacc.c[5] += t6 - t5;
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    using I8 = std::integral_constant<int, K>;
    const int full_hi = (len - 1 - K >= 0) ? (len - 1 - K) / (K + 1) : 0;
    const int interior_end = full_hi + 1;  // blocks [1, full_hi] are interior
    block(0, I8{}, T_{});
    // interior blocks with the unit width as a compile-time constant (one loop body per width)
    dispatch_width<K, kb_min(K)>(Kb, [&](auto kb_c) {
      for (int b = 1; b < interior_end; ++b) block(b, kb_c, F_{});
    });
    for (int b = max(1, interior_end); b < nblk; ++b) block(b, I8{}, T_{});
    trace_unit(P.trace, warp, jr, tile, p0, Kb, src, dst, tacc);
    };
    if constexpr (SCALED_ANY) {
      if (__ldg(P.unsafe + part * (P.ua + 1) + iu) == 0u)
        unit_body(std::true_type{});
      else
        unit_body(std::false_type{});
    } else {
      unit_body(std::false_type{});
    }
  }
}

// Right side: the original per-block protocol (generic-pointer output, lane-0 branches);
// it schedules the unrolled body better than the lean protocol under the 128-register
// budget of 16-warp CTAs.
template <typename T, int K, int R, bool STRICT, bool REFL, bool SCALED_ANY, bool HS, bool LEFT,
          int CDQ = RS_COEF_QUEUE>
__device__ __forceinline__ void pipeline_units_right(const PipeParams& P, unsigned char* smem_raw) {
  static_assert(!LEFT, "right-side protocol");
  constexpr int TR = 32 * R;
  constexpr int CHUNK = (K + 1) * TR;  // ring chunk: K+1 columns x TR owners
  constexpr size_t CBUF = coef_buf_bytes<T, REFL, K>();  // one coefficient buffer (bytes)
  constexpr int S = stages_for(sizeof(T));
  constexpr int FA = S - 1;  // self-fill distance in chunks
  static_assert(FA == 1 || FA == 2, "ring depth must be 2 or 3 chunks");
  constexpr int NBAR = ctl_words(S, LEFT);

  const int NW = P.nw;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  T* ring_sm = reinterpret_cast<T*>(smem_raw + (size_t)NW * 2 * coef_blocks_per_buf(LEFT) * CBUF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring_sm + (size_t)NW * S * CHUNK);

  T* const A = reinterpret_cast<T*>(P.A);
  const int len = P.len;
  const int k = P.k;
  const int nchunk = P.nchunk;
  const int nblk = P.nblk;
  const uint32_t credit = (uint32_t)P.credit;
  constexpr int FB = full_bars(S, false);
  constexpr int SUB = kSub;
  // in-ring of this warp: full[S][SUB], consumed, coef[2]
  uint64_t* const bar_in = bars + warp * NBAR;
  uint64_t* const full_in = bar_in;
  uint32_t* const consumed_in = reinterpret_cast<uint32_t*>(bar_in + FB);
  uint64_t* const cbar = bar_in + FB + 1;
  // position p of a round runs on warp p % NW; the next position on warp + 1
  const int slot = warp;
  uint64_t* const full_out = bars + (warp + 1) * NBAR;
  const uint32_t* const consumed_out = reinterpret_cast<const uint32_t*>(full_out + FB);
  T* const rin = ring_sm + (size_t)warp * S * CHUNK;
  T* const rout = ring_sm + (size_t)(warp + 1) * S * CHUNK;
  unsigned char* const cbuf = smem_raw + (size_t)warp * 2 * coef_blocks_per_buf(LEFT) * CBUF;

  const CtaRange cr = cta_range(P.units, blockIdx.x, gridDim.x, P.t1, P.ua, k, P.sweep_off);
  const long long npos = cr.g1 - cr.g0;
  uint32_t cseq = 0;  // coefficient block pairs consumed by this warp (buffer = cseq&1)

  for (int jr = 0;; ++jr) {
    const long long pos = (long long)jr * NW + slot;
    if (pos >= npos) break;
    const long long g = pos_to_unit(cr, pos);
    const Unit un = unit_at(g, P.t1, P.ua, k, P.sweep_off);
    const long long tile = un.tile;
    const int p0 = un.p0;
    const int Kb = un.kb;
    // the producer of this unit is unit g-1 (same tile, ends at sweep p0); its consumer is
    // g+1. Ring hand-off when that unit is the neighbouring position of the same round.
    int src = SRC_GLOBAL, dst = DST_GLOBAL;
    if (p0 > 0) {
      src = SRC_FLAG;
      if (slot > 0 && g - 1 >= cr.g0 && unit_to_pos(cr, g - 1) == pos - 1) src = SRC_RING;
    }
    if (p0 + Kb < k) {
      dst = DST_FLAG;
      if (slot < NW - 1 && g + 1 < cr.g1 && unit_to_pos(cr, g + 1) == pos + 1) dst = DST_RING;
    }
    const bool self = src != SRC_RING;
    // arithmetic form of this unit: the scaled (fast Givens) records unless the pack
    // flagged this unit's coefficients as outside the scaled form's safe range
    const int part = tile < P.t1 ? 1 : 0;
    const long long iu = g - tile_first_unit(tile, P.t1, P.ua);
    auto unit_body = [&](auto scaled_c) {
    constexpr bool SCALED = decltype(scaled_c)::value;
    using CoefT = std::conditional_t<SCALED, SCoef<T>, Coef<T, REFL>>;

    T* grow[R];        // element (row r, column 0) of this lane's lines
    long long gcs[R];  // column stride; 0 for rows past the matrix (they use the trash slot)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long o = tile * TR + lane + 32 * r;
      const bool ok = o < P.owners;
      grow[r] = ok ? A + o * P.os : reinterpret_cast<T*>(P.trash) + lane + 32 * r;
      gcs[r] = ok ? P.cs : 0;
    }
    // LEFT coalesced chunk copies: this lane's first element e = lane is owner lo0, column
    // lv0; each step of 32 elements advances 3 owners + 5 columns (wrapping past K+1)
    static_assert(!LEFT || 32 == 3 * (K + 1) + 5, "coalesced owner-major copy assumes K + 1 = 9");
    const int lo0 = lane / (K + 1), lv0 = lane - lo0 * (K + 1);
    const long long lstep = 3 * P.os + (32 - 3 * (K + 1)) * P.cs;
    const long long lwrap = P.os - (K + 1) * P.cs;
    const T* const lbase = A + (tile * TR + lo0) * P.os + lv0 * P.cs;
    const bool lfull = tile * TR + TR <= P.owners;
    // this unit's coefficient blocks, contiguous per block (rs_pack_kernel: Kb*(K+1)
    // records; rs_pack_scaled_kernel: Kb*(K+1) records + SR records of scales)
    constexpr int SR = scale_recs(K, sizeof(T));
    const int brec = recs_per_wave(Kb, kPairRecs<T, REFL>) * (K + 1) + (SCALED ? SR : 0);
    const CoefT* ubase;
    if constexpr (SCALED) {
      ubase = reinterpret_cast<const CoefT*>(P.coef_scaled) + (size_t)part * k * nblk * (K + 1 + SR) +
              (size_t)p0 * nblk * (K + 1) + (size_t)iu * nblk * SR;
    } else {
      ubase = reinterpret_cast<const CoefT*>(P.coef) + (size_t)part * k * nblk * (K + 1) + (size_t)p0 * nblk * (K + 1);
    }
    const uint32_t blk_bytes = (uint32_t)(brec * sizeof(CoefT));
    // one elected lane: WAR fence for the buffer's previous readers, arm, start the copy
    // coefficient blocks travel in pairs (blocks 2i, 2i+1: one bulk copy, one wait per two
    // blocks); pair i goes to buffer (cseq + i) & 1
    auto issue_coef = [&](int b, uint32_t buf) {
      if (lane == 0) {
        uint64_t* bar = &cbar[buf];
        const uint32_t bytes = (b + 1 < nblk ? 2u : 1u) * blk_bytes;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, bytes);
        bulk_g2s_nowait(cbuf + (size_t)buf * coef_blocks_per_buf(LEFT) * CBUF, ubase + (size_t)b * brec, bytes, bar);
      }
    };
    const uint32_t seq0 = (uint32_t)jr * (uint32_t)nchunk;
    const uint32_t* myflag = P.flags + tile * k + p0;
    uint32_t* const outflag = P.flags + tile * k + p0 + Kb;
    TraceAcc tacc;
    tacc.t0 = trace_gtime();

    issue_coef(0, cseq & 1);

    // self-filled input (sweep 0 reads A; a flag hand-off reads A after the producer's
    // progress flag): cp.async (LDGSTS) straight into this warp's own ring, FA chunks ahead.
    uint32_t flag_seen = 0;
    auto fill_chunk = [&](int q) {
#ifdef RS_X_NOFILL
      if (src == SRC_GLOBAL) { cp_async_commit(); return; }
#endif
      if (src == SRC_FLAG && flag_seen < (uint32_t)q + 1) flag_seen = wait_flag(myflag, (uint32_t)q + 1);
      if (HS && src == SRC_GLOBAL) {  // host streaming: wait for the copy of these columns
        long long cend = (long long)q * (K + 1) + K;
        if (cend > len - 1) cend = len - 1;
        const uint32_t need = (uint32_t)(cend / P.cw) + 1u;
        if (flag_seen < need) flag_seen = wait_flag(P.arrived, need);
      }
      T* dstp = rin + ((seq0 + (uint32_t)q) % S) * CHUNK;
      const long long c0 = (long long)q * (K + 1);
      if constexpr (LEFT) {
        // owner-major chunk [TR owners][K+1 columns]: element e = i*32 + lane is owner
        // e/(K+1), column e%(K+1) — consecutive lanes read consecutive columns of one owner
        // (contiguous in A on the left side) and write consecutive shared words. (owner,
        // column) and the address advance incrementally (e += 32: +3 owners, +5 columns).
        int v = lv0;
        const T* sp = lbase + c0 * P.cs;
        if (lfull && c0 + K < len) {
#pragma unroll
          for (int i = 0; i < R * (K + 1); ++i) {
            cp_async_elem(dstp + i * 32 + lane, sp, true);
            v += 32 - 3 * (K + 1);
            sp += lstep;
            if (v >= K + 1) v -= K + 1, sp += lwrap;
          }
        } else {
          int ol = lo0;
#pragma unroll
          for (int i = 0; i < R * (K + 1); ++i) {
            const bool ok = tile * TR + ol < P.owners && c0 + v < len;
            cp_async_elem(dstp + i * 32 + lane, ok ? sp : A, ok);
            v += 32 - 3 * (K + 1);
            ol += 3;
            sp += lstep;
            if (v >= K + 1) v -= K + 1, ++ol, sp += lwrap;
          }
        }
        cp_async_commit();
        return;
      }
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
    unsigned long long tc = trace_clock();
    if (self) {
      fill_chunk(0);
      if (FA >= 2 && 1 < nchunk) fill_chunk(1);
      if (FA >= 2 && 1 < nchunk)
        cp_async_wait_group<1>();
      else
        cp_async_wait_group<0>();
      __syncwarp();
      if (lane == 0)
#pragma unroll
        for (int h = 0; h < SUB; ++h) mbar_arrive(&full_in[(seq0 % S) * SUB + h]);
    }
    tacc.c[0] += trace_clock() - tc;

    T w[R][K + 1];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int s = 0; s <= K; ++s) w[r][s] = T(0);

    const bool outring = dst == DST_RING;
    int done_sig = 0;  // host streaming: chunks already released by this (final) unit
    // One block: protocol + compute. KB / EDGE are compile-time so the interior loop
    // carries no per-block branches beyond this unit's hand-off protocol.
    auto block = [&](int b, auto kb_c, auto edge_c, auto first_c) {
      constexpr int KB = decltype(kb_c)::value;
      constexpr bool EDGE = decltype(edge_c)::value;
      constexpr bool FIRST = decltype(first_c)::value;
      unsigned long long t0 = trace_clock();
      const bool pair_start = (b & 1) == 0;
      if (pair_start && b + 2 < nblk) issue_coef(b + 2, (cseq + 1) & 1);
      const bool has_in = !EDGE || b < nchunk;
      const bool has_out = !EDGE || b >= 1;
      if (self && b + FA < nchunk) fill_chunk(b + FA);
      unsigned long long t1 = trace_clock();
      const uint32_t iseq = seq0 + (uint32_t)b;
      const T* islot = rin + (iseq % S) * CHUNK;
      const uint32_t oseq = seq0 + (uint32_t)b - 1u;
      // output pointers: the consumer's ring slot (column stride TR) or A (stride gcs)
      T* op[R];
      long long ostr[R];
      // LEFT, output to A: stage the outgoing chunk in the input slot just read (the last
      // block, which has no input, reuses the previous block's slot) and copy it out below
      T* stage = const_cast<T*>(b < nchunk ? islot : rin + ((iseq - 1u) % S) * CHUNK);
      if (LEFT && outring) {
        T* oslot = rout + (oseq % S) * CHUNK;
#pragma unroll
        for (int r = 0; r < R; ++r) op[r] = oslot + (lane + 32 * r) * (K + 1), ostr[r] = 1;
      } else if (LEFT) {
#pragma unroll
        for (int r = 0; r < R; ++r) op[r] = stage + (lane + 32 * r) * (K + 1), ostr[r] = 1;
      } else if (outring) {
        T* oslot = rout + (oseq % S) * CHUNK + lane;
#pragma unroll
        for (int r = 0; r < R; ++r) op[r] = oslot + 32 * r, ostr[r] = TR;
      } else {
        const long long cb0 = (long long)b * (K + 1) - (K + 1);
#pragma unroll
        for (int r = 0; r < R; ++r) op[r] = grow[r] + cb0 * gcs[r], ostr[r] = gcs[r];
      }
      if (pair_start) mbar_wait(&cbar[cseq & 1], (cseq >> 1) & 1u);
      unsigned long long t2 = trace_clock();
#ifndef RS_X_NOSYNC
      if (!self && has_in) mbar_wait(&full_in[(iseq % S) * SUB], (iseq / S) & 1u);
#endif
      unsigned long long t3 = trace_clock();
      // ring credit: the producer runs at most `credit` chunks ahead of its consumer
#ifndef RS_X_NOSYNC
      if (outring && has_out && oseq >= credit) wait_count(consumed_out, oseq - credit + 1u);
#endif
      unsigned long long t4 = trace_clock();
      {
        const CoefT* cbp =
            reinterpret_cast<const CoefT*>(cbuf + (cseq & 1) * coef_blocks_per_buf(LEFT) * CBUF + (b & 1) * blk_bytes);
        // ring output by STS (default) or through the generic store path shared with A
        // outputs (P.ring_sts = 0: one loop body per unit width)
        uint64_t* const sub_in = (SUB > 1 && !self && has_in) ? &full_in[(iseq % S) * SUB] : nullptr;
        uint64_t* const sub_out = (SUB > 1 && outring && has_out) ? &full_out[(oseq % S) * SUB] : nullptr;
        const uint32_t sub_par = (iseq / S) & 1u;
        if (outring && P.ring_sts) {
#if RS_STS_DIRECT
          // the consumer's ring slot addressed from the shared window itself (not through
          // op[], which also holds global pointers): plain STS with shared-space alias info
          T* const obase_s = rout + (oseq % S) * CHUNK + lane;
#else
          T* const obase_s = op[0];
#endif
          // the draining last block signals the consumer at its final column and stops there
          uint64_t* const early = (SUB == 1 && b == nblk - 1) ? &full_out[oseq % S] : nullptr;
          run_block<T, K, R, KB, STRICT, REFL, EDGE, SCALED, LEFT, true, FIRST, CDQ>(
              w, cbp, islot, op, ostr, obase_s, b, len, Kb, lane, b < nchunk, b >= 1, sub_in, sub_par, sub_out,
              b == nblk - 1, early);
        } else {
          run_block<T, K, R, KB, STRICT, REFL, EDGE, SCALED, LEFT, false, FIRST, CDQ>(
              w, cbp, islot, op, ostr, nullptr, b, len, Kb, lane, b < nchunk, b >= 1, sub_in, sub_par, sub_out,
              b == nblk - 1, nullptr);
        }
      }
      __syncwarp();
      if (LEFT && !outring && has_out) {  // copy the staged chunk to A, columns contiguous
        const long long cb0 = (long long)(b - 1) * (K + 1);
        int v = lv0;
        T* dp = const_cast<T*>(lbase) + cb0 * P.cs;
        if (lfull && cb0 + K < len) {
#pragma unroll
          for (int i = 0; i < R * (K + 1); ++i) {
            *dp = stage[i * 32 + lane];
            v += 32 - 3 * (K + 1);
            dp += lstep;
            if (v >= K + 1) v -= K + 1, dp += lwrap;
          }
        } else {
          int ol = lo0;
#pragma unroll
          for (int i = 0; i < R * (K + 1); ++i) {
            if (tile * TR + ol < P.owners && cb0 + v < len) *dp = stage[i * 32 + lane];
            v += 32 - 3 * (K + 1);
            ol += 3;
            dp += lstep;
            if (v >= K + 1) v -= K + 1, ++ol, dp += lwrap;
          }
        }
        __syncwarp();
      }
      unsigned long long t5 = trace_clock();
      if (lane == 0) {
        // LEFT global output: the last block stages in the slot of chunk nchunk-1, so that
        // slot is released one block later (as nchunk, i.e. iseq of the last block)
        if (LEFT && !outring) {
          if (has_in && b + 1 < nchunk) st_release_shared(consumed_in, iseq + 1u);
          if (b == nchunk) st_release_shared(consumed_in, iseq);
        } else if (has_in) {
          st_release_shared(consumed_in, iseq + 1u);
        }
        // (the last block signalled from inside run_block, at its final column)
        if (SUB == 1 && outring && has_out && !(P.ring_sts && b == nblk - 1)) mbar_arrive(&full_out[oseq % S]);
        if (dst == DST_FLAG && has_out &&
            (b < 2 * kFlagEvery || (b & (kFlagEvery - 1)) == 0 || b >= nblk - RS_FLAG_TAIL)) {
          // the warp barrier above orders every lane's stores before lane 0's gpu-scope
          // fence; the release store then publishes "chunks 0..b-1 are in A"
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          st_release(outflag, (uint32_t)b);
        }
        if (HS && dst == DST_GLOBAL && has_out) {  // host streaming: release finished chunks
          long long e = (long long)b * (K + 1) - 1;  // last column emitted by this block
          if (e > len - 1) e = len - 1;
          const int nd = e == len - 1 ? P.ncw : (int)((e + 1) / P.cw);
          if (nd > done_sig) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (; done_sig < nd; ++done_sig) atomicAdd(P.done + done_sig, 1u);
          }
        }
      }
      if (self && b + 1 < nchunk) {  // the chunk read by the next block has landed
        if (FA >= 2 && b + 2 < nchunk)
          cp_async_wait_group<1>();
        else
          cp_async_wait_group<0>();
        __syncwarp();
        if (lane == 0)
#pragma unroll
          for (int h = 0; h < SUB; ++h) mbar_arrive(&full_in[((iseq + 1u) % S) * SUB + h]);
      }
      if ((b & 1) == 1 || b + 1 == nblk) ++cseq;
      unsigned long long t6 = trace_clock();
      tacc.c[0] += t1 - t0;
      tacc.c[1] += t2 - t1;
      tacc.c[2] += t3 - t2;
      tacc.c[3] += t4 - t3;
      tacc.c[4] += t5 - t4;
      tacc.c[5] += t6 - t5;
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    using I8 = std::integral_constant<int, K>;
    const int full_hi = (len - 1 - K >= 0) ? (len - 1 - K) / (K + 1) : 0;
    const int interior_end = full_hi + 1;  // blocks [1, full_hi] are interior
    // block 0: the compile-time triangle when chunk 0 and block 1 lie inside the matrix
    if (interior_end > 1)
      block(0, I8{}, T_{}, T_{});
    else
      block(0, I8{}, T_{}, F_{});
    // interior blocks with the unit width as a compile-time constant (one loop body per width)
    dispatch_width<K, kb_min(K)>(Kb, [&](auto kb_c) {
      for (int b = 1; b < interior_end; ++b) block(b, kb_c, F_{}, F_{});
    });
    for (int b = max(1, interior_end); b < nblk; ++b) block(b, I8{}, T_{}, F_{});
    trace_unit(P.trace, warp, jr, tile, p0, Kb, src, dst, tacc);
    };
    if constexpr (SCALED_ANY) {
      if (__ldg(P.unsafe + part * (P.ua + 1) + iu) == 0u)
        unit_body(std::true_type{});
      else
        unit_body(std::false_type{});
    } else {
      unit_body(std::false_type{});
    }
  }
}


// HS: host-streaming variant (rs_apply_host_*), a separate instantiation so the resident
// path carries none of its checks. MW: the CTA size the register budget is set for (launch
// bounds): plans of <= 12 warps run a 12-warp build (168 registers per thread instead of
// 128: measured 18.2 -> 18.8 TF/s at config 2, 128 CTAs x 12 warps).
template <typename T, int K, int R, bool STRICT, bool REFL, bool HS, bool LEFT, int MW = max_warps_for(sizeof(T), LEFT, K)>
__global__ void __launch_bounds__(MW * 32, 1) rs_pipeline_kernel(const __grid_constant__ PipeParams P) {
  constexpr int S = stages_for(sizeof(T));
  constexpr int NBAR = ctl_words(S, LEFT);
  constexpr size_t CBUF = coef_buf_bytes<T, REFL, K>();
  // the 168-register build (fp64 right side, <= 12 warps) affords a deeper coefficient queue
  constexpr int CDQ = (sizeof(T) == 8 && !LEFT && MW <= 12 && K == kK) ? RS_COEF_QUEUE_SMALL : RS_COEF_QUEUE;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int NW = P.nw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)NW * 2 * coef_blocks_per_buf(LEFT) * CBUF +
                                               (size_t)NW * S * (K + 1) * 32 * R * sizeof(T));
  // "full" is alias-safe as an mbarrier (the consumer has always seen chunk seq-S before it
  // waits for seq); "consumed" is a monotonic counter because a ring's producer changes
  // between rounds (previous warp vs. self-fill), which a parity test cannot express.
  if (threadIdx.x < NW) {
    uint64_t* bw = bars + threadIdx.x * NBAR;
    constexpr int FB = full_bars(S, LEFT);
#pragma unroll
    for (int i = 0; i < FB; ++i) mbar_init(bw + i, 1);
    *reinterpret_cast<volatile uint32_t*>(bw + FB) = 0u;
    mbar_init(bw + FB + 1, 1);
    mbar_init(bw + FB + 2, 1);
  }
  __syncthreads();
  // fast mode: every unit runs the scaled form unless the pack flagged its coefficients
  // (per unit, P.unsafe) as outside the scaled form's safe range; strict: standard records
  if constexpr (!STRICT) {
    if (P.use_scaled) {
      if constexpr (LEFT || RS_RIGHT_LEAN) {
        pipeline_units<T, K, R, STRICT, REFL, true, HS, LEFT>(P, smem_raw);
      } else {
        pipeline_units_right<T, K, R, STRICT, REFL, true, HS, LEFT, CDQ>(P, smem_raw);
      }
      return;
    }
  }
  if constexpr (LEFT || RS_RIGHT_LEAN) {
    pipeline_units<T, K, R, STRICT, REFL, false, HS, LEFT>(P, smem_raw);
  } else {
    pipeline_units_right<T, K, R, STRICT, REFL, false, HS, LEFT, CDQ>(P, smem_raw);
  }
}

// ------------------------------------------------------------------------------------
// coefficient repack: C/S (len-1) x k column-major -> per-unit blocks. For each sweep
// partition (part 0: ua units per tile, part 1: ua+1), unit i (sweeps p0..p0+kb-1) owns
// nblk blocks of (K+1) x kb records at record offset part*k*nblk*(K+1) + p0*nblk*(K+1):
// block b, wave u, lane l holds rotation (j = b(K+1)+u-1-l, p0+l), zero outside
// 0 <= j <= len-2 — the GPU analogue of the reference's per-window coefficient gather
// (blocking.py:364-373). One bulk copy stages a block. Reverse order mirrors j and
// negates S (rotation) or C (reflector): both exact in IEEE arithmetic.
// ------------------------------------------------------------------------------------
template <typename T, bool REFL, int K>
__global__ void __launch_bounds__(256) rs_pack_kernel(Coef<T, REFL>* __restrict__ out, const T* __restrict__ C,
                                                      const T* __restrict__ Sm, long long ldcs, int len, int k,
                                                      int nblk, int ua, int nparts, int rev,
                                                      const uint32_t* __restrict__ only_if_unsafe, int off) {
  const int per_p = nblk * (K + 1);
  for (int row = blockIdx.y; row < nparts * k; row += gridDim.y) {
    const int part = row / k;
    const int p = row - part * k;
    const int ut = ua + part;
    // unit i of this partition holding sweep p: p0(i) = floor(i*k/ut)
    int i = (int)(((long long)p * ut) / k);
    while (i + 1 < ut && sweep_start(i + 1, ut, k, off) <= p) ++i;
    while (i > 0 && sweep_start(i, ut, k, off) > p) --i;
    // fast mode packs the scaled records first; the standard records are only the
    // fallback of the units whose coefficients are outside the scaled form's safe range
    if (only_if_unsafe != nullptr && only_if_unsafe[part * (ua + 1) + i] == 0u) continue;
    const int p0 = sweep_start(i, ut, k, off);
    const int kb = sweep_start(i + 1, ut, k, off) - p0;
    const int l = p - p0;
    constexpr bool PAIR = kPairRecs<T, REFL>;
    const int nr = recs_per_wave(kb, PAIR);
    Coef<T, REFL>* dst = out + (size_t)part * k * per_p + (size_t)p0 * per_p + (PAIR ? l / 2 : l);
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < per_p; x += gridDim.x * blockDim.x) {
      const int b = x / (K + 1);
      const int u = x - b * (K + 1);
      const long long j = (long long)b * (K + 1) + u - 1 - l;
      Coef<T, REFL> cf{};
      if (j >= 0 && j <= len - 2) {
        const long long jj = rev ? (long long)(len - 2) - j : j;
        T c = __ldg(C + jj + (long long)p * ldcs);
        T s = __ldg(Sm + jj + (long long)p * ldcs);
        if constexpr (REFL) {
          if (rev) c = -c;
          cf.s = s;
          cf.d = c - s;
          cf.e = c + s;
        } else {
          if (rev) s = -s;
          cf.c = c;
          cf.s = s;
        }
      }
      if constexpr (PAIR) {
        T* h = reinterpret_cast<T*>(dst + ((size_t)b * (K + 1) + u) * nr) + 2 * (l & 1);
        h[0] = cf.c;
        h[1] = cf.s;
      } else {
        dst[((size_t)b * (K + 1) + u) * kb] = cf;
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// scaled ("fast Givens") repack for fast-mode fp64. Inside a unit every column j carries a
// scale sigma_j (1 at unit entry) and the window holds x~ = x / sigma. With (c, s) in
// forward form, rotation (j, p) is
//   x' = c*x + s*y = c*sx * (x~ + tau1*y~),  tau1 = s*sy / (c*sx),   sx' = c*sx
//   y' = c*y - s*x = c*sy * (y~ - tau2*x~),  tau2 = s*sx / (c*sy),   sy' = c*sy
// (reflector: y' = s*x - c*y, same taus, sy' = -c*sy), i.e. 2 FMAs instead of 2 MUL +
// 2 FMA. The scales depend only on C/S, so they are computed here, once per call:
// thread (partition, unit, column j) walks the unit's sweeps in application order
// (rotation (j-1, p) before (j, p) before (j+1, p)). The column's final scale is applied
// when the kernel emits it. Records: (tau1, -tau2) at [b][u*kb + l] as in rs_pack_kernel,
// then the K+1 emission scales of the block. A coefficient that would push a scale or tau
// outside [2^-256, 2^256] (or c == 0) flags its unit, unsafe[part*(ua+1) + i]: that unit
// (in every tile) runs the standard form, the other units keep the scaled one.
// ------------------------------------------------------------------------------------
template <typename T, bool REFL, int K>
__global__ void __launch_bounds__(256) rs_pack_scaled_kernel(SCoef<T>* __restrict__ out, const T* __restrict__ C,
                                                             const T* __restrict__ Sm, long long ldcs, int len, int k,
                                                             int nblk, int ua, int nparts, int rev,
                                                             uint32_t* __restrict__ unsafe, int off) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= len) return;
  // scales and taus are formed in fp64 (for fp32 too) and rounded once when stored
  auto coef = [&](int jj, int p, double& c, double& s) {  // forward-form (c, s) of rotation (jj, p)
    const long long jr = rev ? (long long)(len - 2 - jj) : (long long)jj;
    c = (double)C[jr + (long long)p * ldcs];
    s = (double)Sm[jr + (long long)p * ldcs];
    if (rev) {
      if constexpr (REFL) {
        c = -c;
      } else {
        s = -s;
      }
    }
  };
  // safe range of scales / taus: |x~| = |x| / sigma stays far from overflow
  // (fp64: |A| < 2^700; fp32: |A| < 2^60) and no tau overflows the working type
  const double lo = sizeof(T) == 8 ? 0x1p-256 : 0x1p-60, hi = sizeof(T) == 8 ? 0x1p256 : 0x1p60;
  for (int row = blockIdx.y; row < nparts * (ua + 1); row += gridDim.y) {
    const int part = row / (ua + 1);
    const int i = row - part * (ua + 1);  // unit index within the tile
    const int ut = ua + part;
    if (i >= ut) continue;
    const int p0 = sweep_start(i, ut, k, off);
    const int kb = sweep_start(i + 1, ut, k, off) - p0;
    constexpr bool PAIR = kPairRecs<T, REFL>;
    const int nr = recs_per_wave(kb, PAIR);
    constexpr int SR = scale_recs(K, sizeof(T));
    const int brec = nr * (K + 1) + SR;
    SCoef<T>* ubase = out + (size_t)part * k * nblk * (K + 1 + SR) + (size_t)p0 * nblk * (K + 1) +
                      (size_t)i * nblk * SR;
    // the unit's coefficients of rotations (j-1, p), (j, p), (j+1, p), loaded up front
    // (independent loads in flight together; only c is needed for the neighbours)
    double cl[K], cj[K], sj[K], cr[K];
#pragma unroll
    for (int l = 0; l < K; ++l) {
      cl[l] = cj[l] = cr[l] = 1.0;
      sj[l] = 0.0;
      if (l < kb) {
        double sd;
        if (j >= 1) coef(j - 1, p0 + l, cl[l], sd);
        if (j <= len - 2) coef(j, p0 + l, cj[l], sj[l]);
        if (j + 1 <= len - 2) coef(j + 1, p0 + l, cr[l], sd);
      }
    }
    // running scales of columns j and j+1 (a short multiply chain), then the taus of all
    // kb rotations independently (their divisions overlap)
    double sal[K], sbl[K];
    double sa = 1, sb = 1;
    bool bad = false;
#pragma unroll
    for (int l = 0; l < K; ++l) {
      if (l < kb) {
        if (j >= 1) sa *= REFL ? -cl[l] : cl[l];  // rotation (j-1, p) touched column j as its y
        sal[l] = sa;
        sbl[l] = sb;
        if (j <= len - 2) {
          sa *= cj[l];
          sb *= REFL ? -cj[l] : cj[l];
          if (j + 1 <= len - 2) sb *= cr[l];  // rotation (j+1, p) touches column j+1 as its x
        }
        bad |= !(fabs(sa) >= lo && fabs(sa) <= hi) || !(fabs(sb) >= lo && fabs(sb) <= hi);
      }
    }
#pragma unroll
    for (int l = 0; l < K; ++l) {
      if (l < kb && j <= len - 2) {
        const double c = cj[l], s = sj[l];
        // tau1 = s*sb / (c*sa), tau2 = s*sa / (c*sb), with one division
        const double q = 1.0 / (c * sal[l] * sbl[l]);
        const double t1 = s * sbl[l] * sbl[l] * q;
        const double t2 = s * sal[l] * sal[l] * q;
        bad |= !(c != 0.0) || !(fabs(t1) <= hi) || !(fabs(t2) <= hi);
        // rotation (j, p) runs in block b at wave u with b(K+1) + u = j + 1 + l
        const int bu = j + 1 + l;
        const int b = bu / (K + 1), u = bu - b * (K + 1);
        SCoef<T> rec{};
        rec.c = (T)t1;
        rec.s = (T)-t2;
        if constexpr (PAIR) {
          T* h = reinterpret_cast<T*>(ubase + (size_t)b * brec + u * nr + l / 2) + 2 * (l & 1);
          h[0] = rec.c;
          h[1] = rec.s;
        } else {
          ubase[(size_t)b * brec + u * kb + l] = rec;
        }
      }
    }
    // column j is emitted at block j/(K+1) + 1, wave j%(K+1)
    const int be = j / (K + 1) + 1, ue = j - (j / (K + 1)) * (K + 1);
    if (be < nblk) reinterpret_cast<T*>(ubase + (size_t)be * brec + (size_t)nr * (K + 1))[ue] = (T)sa;
    if (bad) atomicOr(unsafe + part * (ua + 1) + i, 1u);
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
// micro-kernel API (the reference's kernel_wave_apply, kernels.py:81-103, 335-371): a
// panel of m_r rows, column j at P + j*ld (rows contiguous); wave w, lane l rotates
// columns (col0 + w + KR-1-l, +1) with ct/st[w*KR + l] (wave-major tiles). One thread per
// row. The coefficient tiles are staged through shared memory in chunks of
// kWaveChunkBlocks*(KR+1) waves; each thread keeps the (KR+1)-column window in registers,
// waves unrolled in blocks of KR+1 so the window slots are compile-time (slot = column
// mod (KR+1), the same register residency as the pipeline kernel): every panel element is
// loaded and stored once per call.
// ------------------------------------------------------------------------------------
constexpr int kWaveChunkBlocks = 16;
template <typename T, int KR, bool STRICT, bool REFL>
__global__ void __launch_bounds__(128) rs_wave_kernel(T* __restrict__ P, long long m_r, long long ld,
                                                      const T* __restrict__ ct, const T* __restrict__ st,
                                                      long long n_waves, long long col0) {
  constexpr int M = KR + 1;
  constexpr int CHW = kWaveChunkBlocks * M;  // waves per staged chunk (a multiple of M)
  extern __shared__ __align__(16) unsigned char wave_smem[];
  T* const sc = reinterpret_cast<T*>(wave_smem);
  T* const ss = sc + CHW * KR;
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = row < m_r;
  T* const pr = P + (ok ? row : 0) + col0 * ld;
  T win[M];
  // at the start of wave w the window holds columns [w-1, w+KR-1]; column w+KR enters
#pragma unroll
  for (int c = 0; c < M; ++c) win[c] = (c < KR && ok) ? pr[c * ld] : T(0);
  for (long long w0 = 0; w0 < n_waves; w0 += CHW) {
    const long long nw = n_waves - w0 < CHW ? n_waves - w0 : CHW;
    __syncthreads();
    for (long long i = threadIdx.x; i < nw * KR; i += blockDim.x) {
      sc[i] = ct[w0 * KR + i];
      ss[i] = st[w0 * KR + i];
    }
    __syncthreads();
    for (long long wb = 0; wb < nw; wb += M) {
#pragma unroll
      for (int u = 0; u < M; ++u) {
        const long long w = w0 + wb + u;  // (w0 + wb) % M == 0: slot of column w is u
        if (w < n_waves) {
          win[(u + KR) % M] = ok ? pr[(w + KR) * ld] : T(0);
#pragma unroll
          for (int l = 0; l < KR; ++l) {
            const T c = sc[(wb + u) * KR + l];
            const T s = ss[(wb + u) * KR + l];
            T& x = win[(u + KR - 1 - l) % M];
            T& y = win[(u + KR - l) % M];
            if constexpr (REFL) {
              refl2<T, STRICT>(x, y, s, sub_rn(c, s), add_rn(c, s));
            } else {
              rot2<T, STRICT>(x, y, c, s);
            }
          }
          // column w is final after wave w (its last transform is lane KR-1's x)
          if (ok) pr[w * ld] = win[u];
        }
      }
    }
  }
  // the columns still in the window, [n_waves, n_waves + KR), go back too
  if (ok) {
    const int base = (int)(n_waves % M);
#pragma unroll
    for (int sl = 0; sl < M; ++sl) {
      const long long col = n_waves + (sl - base + M) % M;
      if (col < n_waves + KR) pr[col * ld] = win[sl];
    }
  }
}
// wider waves (KR > 8): the same schedule with the window in L1 (global loads/stores)
template <typename T, bool STRICT, bool REFL>
__global__ void __launch_bounds__(128) rs_wave_kernel_wide(T* __restrict__ P, long long m_r, long long ld,
                                                           const T* __restrict__ ct, const T* __restrict__ st,
                                                           long long n_waves, int k_r, long long col0) {
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m_r) return;
  T* const pr = P + row + col0 * ld;
  for (long long w = 0; w < n_waves; ++w) {
    for (int l = 0; l < k_r; ++l) {
      const long long j = w + k_r - 1 - l;
      const T c = __ldg(ct + w * k_r + l), s = __ldg(st + w * k_r + l);
      T x = pr[j * ld], y = pr[(j + 1) * ld];
      if constexpr (REFL) {
        refl2<T, STRICT>(x, y, s, sub_rn(c, s), add_rn(c, s));
      } else {
        rot2<T, STRICT>(x, y, c, s);
      }
      pr[j * ld] = x;
      pr[(j + 1) * ld] = y;
    }
  }
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

// Launches the pipeline kernel family <T, STRICT, REFL, HS> (defined and explicitly
// instantiated in pipeline_variant.cu, one translation unit per family).
template <typename T, bool STRICT, bool REFL, bool HS, bool LEFT, int K, int MW>
cudaError_t launch_pipeline(const cudaLaunchConfig_t& cfg, const PipeParams& P);
// right-side plans of at most this many warps per CTA use the 168-register build
constexpr int kSmallCtaWarps = 12;

}  // namespace rsk
