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
//   * A "unit" is (tile of 32*R owners, 1..K consecutive sweeps). One warp runs one unit:
//     every lane owns R rows (right side; columns for the left side) and keeps a
//     (K+1)-column window of them in registers. Waves are processed in blocks of K+1 so
//     the window rotates through fixed registers (slot = column mod (K+1)) — true register
//     residency, which the reference only models (SURVEY §2 note, kernels.py:135-147).
//   * Work split: the tile-major sequence of (tile, sweep) pairs is cut into one equal
//     range per SM sub-partition (4 per SM), each range into units of <= K sweeps with
//     compile-time widths. Every SMSP therefore carries the same FP64 work, whatever the
//     shape (the reference splits rows over threads, blocking.py:518-526).
//   * Consecutive units of one tile are chained warp-to-warp (same sub-partition) through
//     shared-memory rings guarded by an mbarrier (full) and a monotonic counter (consumed),
//     so A crosses HBM once per chain instead of once per unit. A chain that crosses a
//     sub-partition or round boundary is handed off through A itself (in place) with
//     release/acquire progress flags in global memory. All CTAs are co-resident
//     (cooperative launch), so waits always make progress.
//   * Coefficients are repacked once per call into sweep-major rows of (c,s) records padded
//     on both sides (the GPU analogue of the reference's per-window coefficient gather,
//     blocking.py:364-373). Per block each of the unit's lanes stages its K+1 records with a
//     cp.async.bulk (TMA bulk copy) into a per-warp double buffer; every thread reads them
//     as broadcast LDS.128.
//   * strict mode uses __dmul_rn/__dadd_rn/__dsub_rn in the reference's exact expression
//     shape (no contraction => bit-identical to the reference strict build); fast mode uses
//     2 DMUL + 2 DFMA per rotation element (the 4-instruction minimum for 6 flops).

#include <cuda.h>  // stream memory-op types (entry points resolved at run time)
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "rotseq_b200.h"
#include "rotseq_device.cuh"

#define RS_VERSION 10300

namespace rsk {
// the FP64 tensor-core variant (dmma_variant.cu)
size_t dmma_workspace(int64_t m, int64_t n, int64_t k);
int dmma_run(double* A, int64_t m, int64_t n, int64_t lda, const double* C, const double* S, int64_t ldcs,
             int64_t k, int rev, int refl, void* workspace, cudaStream_t st);
}  // namespace rsk

namespace {

using namespace rsk;

std::atomic<long long> g_launches{0};
thread_local std::string g_err;
unsigned long long* g_trace_buf = nullptr;  // rs_debug_set_trace (RS_TRACE builds)

rs_status fail(rs_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

// ------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------
struct Geometry {
  long long owners = 0;
  int len = 0;
  long long os = 0, cs = 0;
  int k = 0;
  long long tiles = 0;
  long long pairs = 0;  // (tile, sweep) pairs = tiles * k
  int nchunk = 0;
  int nblk = 0;
  int kw = kK;  // sweeps per unit window: kK, or wide_k (right side, units of >= 9 sweeps)
  size_t coef_rec = 0;
  size_t std_bytes = 0;     // standard records (both sweep partitions)
  size_t coef_bytes = 0;    // standard + scaled records
  size_t flags_only = 0;    // progress flags (zeroed per launch)
  size_t unsafe_bytes = 0;  // per-unit "outside the scaled form's range" words, [2][ua+1]
  size_t flag_bytes = 0;    // flags + unsafe words + trash slot
  bool left = false;
  bool refl = false;
  bool streaming = false;  // host streaming (rs_apply_host_*): input-bound, plain plans only
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Library-private stream-ordered pool per device: scratch (workspace, device copies of
// host matrices) is returned to it at the end of each call and reused by the next one
// instead of being unmapped at every synchronisation (release threshold 2 GiB; the default
// pool's threshold of 0 made every rs_apply_host_* call map ~150 MB afresh).
cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && pools[dev] == nullptr) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      cudaMemPool_t np = nullptr;
      if (cudaMemPoolCreate(&np, &props) == cudaSuccess) {
        uint64_t thr = 2ull << 30;
        cudaMemPoolSetAttribute(np, cudaMemPoolAttrReleaseThreshold, &thr);
        pools[dev] = np;
      } else {
        cudaGetLastError();
      }
    }
    if (dev < 64) pool = pools[dev];
  }
  if (pool == nullptr) return cudaMallocAsync(p, bytes, st);
  return cudaMallocFromPoolAsync(p, bytes, pool, st);
}


bool make_geometry(int64_t m, int64_t n, int64_t lda, int64_t k, int side, int kind, int dtype, Geometry* g) {
  const bool left = side == RS_SIDE_LEFT;
  g->left = left;
  g->refl = kind == RS_KIND_REFLECTOR;
  g->owners = left ? n : m;
  g->len = (int)(left ? m : n);
  g->os = left ? lda : 1;
  g->cs = left ? 1 : lda;
  g->k = (int)k;
  const int towners = tile_owners(dtype == RS_DTYPE_F64 ? 8 : 4);
  g->tiles = (g->owners + towners - 1) / towners;
  g->pairs = g->tiles * g->k;
  // the 16-sweep window: fp32, right side, and every unit of the full-width split at
  // least 9 sweeps wide (the wide kernel is compiled for widths 9..16)
  g->kw = kK;
  const bool f32 = dtype == RS_DTYPE_F32;
  const bool wide_ok = f32 ? (RS_F32_WIDE && !getenv("RS_F32_K8")) : (RS_F64_WIDE && !getenv("RS_F64_K8"));
  const int kwide = wide_k(f32 ? 4 : 8);
  if (wide_ok && !left && k >= kwide) {
    const int64_t ut0 = (k + kwide - 1) / kwide;
    if (k / ut0 >= kb_min(kwide)) g->kw = kwide;
  }
  g->nchunk = (g->len + g->kw) / (g->kw + 1);
  g->nblk = g->nchunk + 1;
  const size_t tsz = dtype == RS_DTYPE_F64 ? 8 : 4;
  g->coef_rec = (kind == RS_KIND_REFLECTOR ? 4 * tsz : 16);
  // two sweep partitions (ua and ua+1 units per tile) of k * nblk * (K+1) records each
  g->std_bytes = align_up(2 * (size_t)g->k * g->nblk * (g->kw + 1) * g->coef_rec, 256);
  // scaled form: per partition k*nblk*(K+1) records + <= k*nblk*SR scale records
  const size_t sr = (size_t)scale_recs(g->kw, f32 ? 4 : 8);
  g->coef_bytes = g->std_bytes + align_up(2 * (size_t)g->k * g->nblk * (g->kw + 1 + sr) * 16, 256);
  g->flags_only = align_up((size_t)(g->pairs + 1) * sizeof(uint32_t), 256);
  g->unsafe_bytes = align_up(2 * (size_t)(g->k + 1) * sizeof(uint32_t), 256);  // ua + 1 <= k + 1
  g->flag_bytes = g->flags_only + g->unsafe_bytes + kTrashBytes;
  return true;
}

struct LaunchPlan {
  int grid = 0;
  int nw = 0;
  size_t smem = 0;
  long long units = 0;
  int ua = 0;
  long long t1 = 0;
  int mode = 1;  // 1: few units per SMSP (mixed widths); 2: full-width units; 3: aligned;
                 // 4: equal chains of mixed widths on more SMs than the aligned plan
  int sweep_off = 0;  // offset of the sweep split (sweep_start)
};

size_t smem_per_warp(size_t tsz, size_t coef_rec, bool left, int K, bool refl) {
  // == coef_buf_bytes<T, REFL, K>() (fp32 rotation records hold two lanes each)
  const size_t cbuf = coef_block_bytes(K, tsz == 4 && !refl, coef_rec, tsz);
  return 2 * coef_blocks_per_buf(left) * cbuf + (size_t)stages_for(tsz) * (K + 1) * tile_owners(tsz) * tsz +
         ctl_words(stages_for(tsz), left) * sizeof(uint64_t);
}

// Grid of G <= #SMs persistent CTAs and U = 4*G*q units (q per SM sub-partition, each
// unit <= K sweeps wide), NW = 4 * ceil(q / rounds) warps per CTA: one round when the q
// units of a sub-partition fit, else the fewest rounds of at most cap/4 warps each.
rs_status plan_launch(const Geometry& g, size_t tsz, LaunchPlan* lp) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(RS_ECUDA, "cudaGetDevice failed");
  int sms = 0, optin = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return fail(RS_ECUDA, "cudaDeviceGetAttribute failed");
  const size_t per = smem_per_warp(tsz, g.coef_rec, g.left, g.kw, g.refl);
  // one extra control block: the (never dereferenced) out-ring words of the last warp
  const size_t ctl = ctl_words(stages_for(tsz), g.left) * sizeof(uint64_t);
  int cap = (int)((optin - ctl) / per);
  const int wmax = max_warps_for(tsz, g.left, g.kw);
  if (cap > wmax) cap = wmax;
  cap &= ~3;
  if (cap < 4) return fail(RS_EUNSUPPORTED, "shared memory too small for one warp per sub-partition");
  long long grid = sms;
  // test hooks: force multi-round / multi-CTA geometry on small problems
  if (const char* ev = getenv("RS_DEBUG_MAX_WARPS")) {
    const int v = atoi(ev);
    if (v >= 1 && v < cap) cap = v < 4 ? 4 : (v & ~3);
  }
  if (const char* ev = getenv("RS_DEBUG_GRID")) {
    const long long v = atoll(ev);
    if (v >= 1 && v < grid) grid = v;
  }
  // Aligned plan: every unit exactly w = k/ut sweeps wide (ut divides k, w <= K), every CTA
  // runs r rounds of nw warps and the tiles' chains of ut units fill CTA rounds exactly
  // (ut % nw == 0 or nw % ut == 0): all chains identical and every sub-partition equally
  // loaded, at the price of idling the SMs left over (G' = #CTAs divides the work; 128 of
  // 148 here). It wins for few rounds (measured, B200: config 2 17.8 -> 18.3 TF/s on 128
  // CTAs x 12 warps; config 4 30.1 -> 31.2; config 5 19.7 -> 21.5; 16384 x 2048 x 256
  // 19.7 -> 21.3) and loses for many (config 3, 16 rounds: 24.2 -> 21.7), so it is used
  // for r <= 4 rounds on >= 80% of the SMs, preferring more CTAs, then wider units.
  const bool hooks = getenv("RS_DEBUG_GRID") || getenv("RS_PLAN_MODE") || getenv("RS_PLAN_Q");
  // (host streaming is input-bound: it keeps every SM, measured 3.61 vs 3.75 ms at config 2)
  if (!hooks && !g.streaming && !getenv("RS_NO_ALIGNED_PLAN")) {
    long long bestG = 0, bestU = 0;
    int bestNW = 0;
    const int ut0 = (g.k + g.kw - 1) / g.kw;
    // developer knobs (measurements): force the chain length / warps per CTA
    const int force_ut = getenv("RS_ALIGNED_UT") ? atoi(getenv("RS_ALIGNED_UT")) : 0;
    const int force_nw = getenv("RS_ALIGNED_NW") ? atoi(getenv("RS_ALIGNED_NW")) : 0;
    for (int ut = ut0; ut <= 2 * ut0 && ut <= g.k; ++ut) {
      if (g.k % ut != 0) continue;
      if (g.k / ut < kb_min(g.kw)) continue;  // wide window: units of >= 9 sweeps only
      if (force_ut > 0 && ut != force_ut) continue;
      const long long U = g.tiles * ut;
      for (int nw = cap; nw >= 8; nw -= 4) {
        if (force_nw > 0 && nw != force_nw) continue;
        if (!(ut % nw == 0 || nw % ut == 0) || U % nw != 0) continue;
        const long long cr = U / nw;  // CTA-rounds
        long long r = (cr + grid - 1) / grid;
        while (r <= 4 && cr % r != 0) ++r;
        if (r > 4) continue;
        const long long G2 = cr / r;
        if (G2 * 5 < grid * 4) continue;
        if (G2 > bestG) bestG = G2, bestU = U, bestNW = nw;
      }
    }
    // Equal-chain plan: when the aligned plan runs a single round on fewer SMs than the
    // device has, chains of ut' > ut units (widths floor/ceil of k/ut', the wider ones placed
    // mid-period by sweep_off = ut'/2, away from the chain's tail and from most flag
    // hand-offs) can fill more SMs with one unit per warp: every chain identical, every
    // sub-partition within one sweep of the others. Taken when the modelled time
    //   (blocks + 2.2 per ring hop + 9 per CTA crossing) x (sweeps per sub-partition)
    // beats the aligned plan's by 2% (measured, B200, config 2: 144 CTAs x 12 warps, 27
    // units of 7-8 sweeps per tile, 19.1 vs 18.7 TF/s; with the wide units last, as
    // sweep_off = 0 puts them, the same plan gives 18.3).
    // Only where the aligned chains already cross CTAs (ut > nw): a chain that fits one
    // CTA has no flag hand-off at all, and giving it some costs more than the extra SMs
    // return (measured, config 4: 30.2 vs 32.9 TF/s).
    // Right side only: the left-side protocol lacks the shorter unit edges and loses with the
    // longer chains (4096^2, k = 192, left / reverse: 16.8 vs 17.6 TF/s).
    if (bestG > 0 && bestG < grid && bestU / bestNW == bestG && bestU / g.tiles > bestNW && !g.left &&
        !getenv("RS_NO_EQUAL_CHAIN")) {
      const int ut_a = (int)(bestU / g.tiles);
      auto cost = [&](int ut, int nw, int per_smsp_sweeps) {
        const double cross = (double)((ut + nw - 1) / nw - 1) + (ut % nw ? 0.5 : 0.0);
        return ((double)g.nblk + 2.2 * (ut - 1) + 9.0 * cross) * per_smsp_sweeps;
      };
      const double cost_a = cost(ut_a, bestNW, (bestNW / 4) * (g.k / ut_a));
      double best_c = 0.98 * cost_a;
      long long eG = 0, eU = 0;
      int eNW = 0;
      // developer knobs (measurements): force the chain length / warps per CTA
      const int force_eut = getenv("RS_EQ_UT") ? atoi(getenv("RS_EQ_UT")) : 0;
      const int force_enw = getenv("RS_EQ_NW") ? atoi(getenv("RS_EQ_NW")) : 0;
      if (force_eut > 0) best_c = 1e300;
      for (int ut = ut_a + 1; (ut <= ut_a + ut_a / 4 || force_eut > 0) && ut <= g.k; ++ut) {
        if (force_eut > 0 && ut != force_eut) continue;
        if (g.k % ut == 0 || g.k / ut < 2) continue;  // uniform widths are the aligned plan's
        const long long U = g.tiles * ut;
        for (int nw = cap; nw >= 8; nw -= 4) {
          if (force_enw > 0 && nw != force_enw) continue;
          if (U % nw != 0) continue;
          const long long G2 = U / nw;
          if (G2 > grid || G2 <= bestG) continue;
          // per sub-partition: nw/4 units of floor(k/ut) sweeps and at most one wider one
          // (the wide units are at least 4 chain positions apart when k % ut <= ut / 4)
          if ((long long)(g.k % ut) * 4 > ut && force_eut == 0) continue;
          const double c = cost(ut, nw, (nw / 4) * (g.k / ut) + 1);
          if (c < best_c) best_c = c, eG = G2, eU = U, eNW = nw;
        }
      }
      if (eG > 0) {
        lp->grid = (int)eG;
        lp->nw = eNW;
        lp->smem = per * eNW + ctl;
        lp->units = eU;
        lp->mode = 4;
        lp->ua = (int)(eU / g.tiles);
        lp->t1 = 0;
        // the offset whose wide units fall least often on a chain's head, tail or flag
        // hand-off units (first / last unit of a CTA's range), over the tiles' phases
        // against the CTA boundaries (config 2: offsets 3-5, wide units at 7, 16, 25 of 27:
        // 19.3 TF/s; 9 -> 18.4, 18 -> 18.6, where they meet the flag units)
        // (memoised: the search is ~9000 steps of host time on every launch otherwise)
        struct OffMemo { int ut = 0, nw = 0, k = 0, off = 0; };
        static thread_local OffMemo memo;
        if (memo.ut == lp->ua && memo.nw == eNW && memo.k == g.k) {
          lp->sweep_off = memo.off;
        } else {
          const int ut = lp->ua, nw = eNW, w0 = g.k / ut;
          int best_off = 0;
          long long best_score = -1;
          for (int off = 0; off < ut; ++off) {
            long long score = 0;
            for (int t = 0; t < nw; ++t) {  // phases repeat with period <= nw tiles
              const int phase = (int)(((long long)t * ut) % nw);
              for (int i = 0; i < ut; ++i) {
                if (sweep_start(i + 1, ut, g.k, off) - sweep_start(i, ut, g.k, off) <= w0) continue;
                const int pos = (phase + i) % nw;
                if (i == 0 || i == ut - 1 || pos == 0 || pos == nw - 1) ++score;
              }
            }
            if (best_score < 0 || score < best_score) best_score = score, best_off = off;
          }
          lp->sweep_off = best_off;
          memo.ut = ut, memo.nw = nw, memo.k = g.k, memo.off = best_off;
        }
        if (const char* ev = getenv("RS_SWEEP_OFF")) {
          const int v = atoi(ev);
          if (v >= 0 && v < lp->ua) lp->sweep_off = v;
        }
        return RS_OK;
      }
    }
    if (bestG > 0) {
      lp->grid = (int)bestG;
      lp->nw = bestNW;
      lp->smem = per * bestNW + ctl;
      lp->units = bestU;
      lp->mode = 3;
      lp->ua = (int)(bestU / g.tiles);
      lp->t1 = 0;
      return RS_OK;
    }
  }
  const long long umin = g.tiles * ((g.k + g.kw - 1) / g.kw);
  const long long gneed = (umin + 3) / 4;
  if (gneed < grid) grid = gneed;
  if (grid < 1) grid = 1;
  long long q = (umin + 4 * grid - 1) / (4 * grid);
  if (const char* ev = getenv("RS_PLAN_Q")) {
    const long long v = atoll(ev);
    if (v > q) q = v;
  }
  // Few units per sub-partition: U = 4*G*q balances every sub-partition exactly (widths
  // k/u_t, mixed). Many units (several rounds): full-width units (U = umin) keep every
  // round's per-SMSP load equal and the residual imbalance (< 1/q) is small.
  // Mode 1 also loses when its extra units barely narrow them (average width > 7.5 of 8):
  // a tile then mixes 7- and 8-wide units and its chain runs at the 8-wide units' pace
  // (measured: 8192 x 2048 x 256, the 8-GPU shard of config 3: 18.9 -> 20.7 TF/s).
  const double w1 = (double)g.k * (double)g.tiles / (double)(4 * grid * q);
  int mode = (q >= 8 || w1 > 7.5) ? 2 : 1;
  if (const char* ev = getenv("RS_PLAN_MODE")) {
    const int v = atoi(ev);
    if (v == 1 || v == 2) mode = v;
  }
  // the wide window runs units of >= 9 sweeps only: full-width units (mode 2) unless
  // the few-units split keeps every unit that wide
  if (g.kw > kK && (double)g.k * g.tiles / (double)(4 * grid * q) < kb_min(g.kw) + 1) mode = 2;
  long long U = mode == 1 ? 4 * grid * q : umin;
  if (U > g.pairs) U = g.pairs;  // at least one sweep per unit
  // the fewest rounds of <= cap warps, spread evenly (equal rounds keep every round's
  // warps per sub-partition, and so its latency hiding, the same)
  const long long nmax = (U + grid - 1) / grid;
  const long long rounds = (nmax + cap - 1) / cap;
  const long long per_round = (nmax + rounds - 1) / rounds;
  int nw = (int)(((per_round + 3) / 4) * 4);
  if (nw > cap) nw = cap;
  lp->grid = (int)grid;
  lp->nw = nw;
  lp->smem = per * nw + ctl;
  lp->units = U;
  lp->mode = mode;
  lp->ua = (int)(U / g.tiles);
  lp->t1 = U % g.tiles;
  return RS_OK;
}

struct HostStream {
  const uint32_t* arrived = nullptr;
  uint32_t* done = nullptr;
  int cw = 1;
  int ncw = 0;
};

template <typename T, bool REFL>
rs_status launch_pack(const Geometry& g, const T* C, const T* S, long long ldcs, int rev, void* ws,
                      cudaStream_t st, bool scaled, bool std_only_if_unsafe = false) {
  using CoefT = Coef<T, REFL>;
  CoefT* coef = reinterpret_cast<CoefT*>(ws);
  LaunchPlan lp;  // the unit partition of the sweeps comes from the launch plan
  rs_status rc = plan_launch(g, sizeof(T), &lp);
  if (rc != RS_OK) return rc;
  const int nparts = lp.t1 > 0 ? 2 : 1;
  const int per_p = g.nblk * (g.kw + 1);
  int bx = (per_p + 255) / 256;
  if (bx > 64) bx = 64;
  const int rows = nparts * g.k;
  // rows are grid-strided: a capped grid keeps the (usual) early exit after the scaled
  // pack cheap (3264 CTAs that only test the unsafe word cost ~4 us at config 2); up to
  // 64 x 32 CTAs of 256 threads still saturate HBM when the standard records are written
  const int by = rows < 32 ? rows : 32;
  // Scaled records first (fast mode); the standard records are the fallback the pipeline
  // uses when the scaled form is out of range, so a per-call pack (std_only_if_unsafe)
  // lets the standard pack kernel exit at once when the scaled records are safe. The
  // resident pack (rs_pack_*) always writes both: strict or fast is chosen per apply.
  uint32_t* unsafe = nullptr;
  if (scaled) {
    unsigned char* base = reinterpret_cast<unsigned char*>(ws);
    unsafe = reinterpret_cast<uint32_t*>(base + g.coef_bytes + g.flags_only);
    cudaError_t e0 = cudaMemsetAsync(unsafe, 0, 2 * (size_t)(lp.ua + 1) * sizeof(uint32_t), st);
    if (e0 != cudaSuccess) return fail(RS_ECUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e0));
    const int srows = nparts * (lp.ua + 1);
    const int sy = srows < 65535 ? srows : 65535;
    const dim3 sgrid((unsigned)((g.len + 127) / 128), (unsigned)sy);
    SCoef<T>* const sout = reinterpret_cast<SCoef<T>*>(base + g.std_bytes);
    if (g.kw == wide_k(sizeof(T)))
      rs_pack_scaled_kernel<T, REFL, wide_k(sizeof(T))><<<sgrid, 128, 0, st>>>(sout, C, S, ldcs, g.len, g.k, g.nblk, lp.ua,
                                                                    nparts, rev, unsafe, lp.sweep_off);
    else
      rs_pack_scaled_kernel<T, REFL, kK><<<sgrid, 128, 0, st>>>(sout, C, S, ldcs, g.len, g.k, g.nblk, lp.ua, nparts,
                                                                rev, unsafe, lp.sweep_off);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  const uint32_t* const only = scaled && std_only_if_unsafe ? unsafe : nullptr;
  if (g.kw == wide_k(sizeof(T)))
    rs_pack_kernel<T, REFL, wide_k(sizeof(T))><<<dim3((unsigned)bx, (unsigned)by), 256, 0, st>>>(coef, C, S, ldcs, g.len, g.k,
                                                                                      g.nblk, lp.ua, nparts, rev, only, lp.sweep_off);
  else
    rs_pack_kernel<T, REFL, kK><<<dim3((unsigned)bx, (unsigned)by), 256, 0, st>>>(coef, C, S, ldcs, g.len, g.k,
                                                                                  g.nblk, lp.ua, nparts, rev, only, lp.sweep_off);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("pack launch: ") + cudaGetErrorString(e));
  return RS_OK;
}

// Runs the pipeline on coefficients already packed into `ws` (by launch_pack with the
// same geometry, order and kind). Resets the hand-off flags first.
bool scaled_disabled() {
  const char* e = getenv("RS_NO_SCALED");
  return e != nullptr && atoi(e) != 0;
}

template <typename T, bool STRICT, bool REFL>
rs_status launch_run(const Geometry& g, T* Abase, int rev, void* ws, cudaStream_t st,
                     const HostStream* hs = nullptr) {
  const int use_scaled = (!STRICT && !scaled_disabled()) ? 1 : 0;
  using CoefT = Coef<T, REFL>;
  LaunchPlan lp;
  rs_status rc = plan_launch(g, sizeof(T), &lp);
  if (rc != RS_OK) return rc;
  CoefT* coef = reinterpret_cast<CoefT*>(ws);
  uint32_t* flags = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(ws) + g.coef_bytes);
  cudaError_t e = cudaMemsetAsync(flags, 0, g.flags_only, st);
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  PipeParams P;
  P.A = Abase;
  P.os = g.os;
  P.cs = rev ? -g.cs : g.cs;
  if (rev) P.A = Abase + (long long)(g.len - 1) * g.cs;
  P.owners = g.owners;
  P.tiles = g.tiles;
  P.units = lp.units;
  P.t1 = lp.t1;
  P.ua = lp.ua;
  P.coef = coef;
  P.flags = flags;
  P.trash = reinterpret_cast<unsigned char*>(ws) + g.coef_bytes + g.flags_only + g.unsafe_bytes;
  P.coef_scaled = reinterpret_cast<unsigned char*>(ws) + g.std_bytes;
  P.unsafe = reinterpret_cast<const uint32_t*>(reinterpret_cast<unsigned char*>(ws) + g.coef_bytes + g.flags_only);
  P.use_scaled = use_scaled;
  P.arrived = hs ? hs->arrived : nullptr;
  P.done = hs ? hs->done : nullptr;
  P.cw = hs ? hs->cw : 1;
  P.ncw = hs ? hs->ncw : 0;
  P.credit = stages_for(sizeof(T));
  P.ring_sts = 1;
  if (const char* ev = getenv("RS_RING_STS")) P.ring_sts = atoi(ev);
  if (const char* ev = getenv("RS_CREDIT")) {
    const int v = atoi(ev);
    if (v >= 1 && v <= stages_for(sizeof(T))) P.credit = v;
  }
  P.sweep_off = lp.sweep_off;
  P.len = g.len;
  P.k = g.k;
  P.nchunk = g.nchunk;
  P.nblk = g.nblk;
  P.nw = lp.nw;
  P.trace = g_trace_buf;
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
  const bool left = g.os != 1;  // owners are columns: owner-major rings, coalesced A I/O
  constexpr size_t TS = sizeof(T);
  constexpr int MWR = max_warps_for(TS, false, kK), MWL = max_warps_for(TS, true, kK);
  // fp64 right side: plans of <= 12 warps per CTA run the 168-register build
  const bool small = TS == 8 && !left && lp.nw <= kSmallCtaWarps && !getenv("RS_NO_SMALL_CTA");
  if (g.kw != kK) {
    constexpr int KW = wide_k(TS);
    if constexpr ((TS == 4 && RS_F32_WIDE) || (TS == 8 && RS_F64_WIDE)) {
      constexpr int MWW = max_warps_for(TS, false, KW);
      if (left || g.kw != KW) return fail(RS_EUNSUPPORTED, "wide window: right-side launches only");
      e = hs ? launch_pipeline<T, STRICT, REFL, true, false, KW, MWW>(cfg, P)
             : launch_pipeline<T, STRICT, REFL, false, false, KW, MWW>(cfg, P);
    } else {
      return fail(RS_EUNSUPPORTED, "wide window not built");
    }
  } else if (left) {
    e = hs ? launch_pipeline<T, STRICT, REFL, true, true, kK, MWL>(cfg, P)
           : launch_pipeline<T, STRICT, REFL, false, true, kK, MWL>(cfg, P);
  } else if (small) {
    if constexpr (TS == 8) {
      e = hs ? launch_pipeline<T, STRICT, REFL, true, false, kK, kSmallCtaWarps>(cfg, P)
             : launch_pipeline<T, STRICT, REFL, false, false, kK, kSmallCtaWarps>(cfg, P);
    }
  } else {
    e = hs ? launch_pipeline<T, STRICT, REFL, true, false, kK, MWR>(cfg, P)
           : launch_pipeline<T, STRICT, REFL, false, false, kK, MWR>(cfg, P);
  }
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
rs_status run_dispatch(const Geometry& g, T* A, int rev, int kind, int strict, void* ws, cudaStream_t st,
                       const HostStream* hs = nullptr) {
  if (strict)
    return kind == RS_KIND_REFLECTOR ? launch_run<T, true, true>(g, A, rev, ws, st, hs)
                                     : launch_run<T, true, false>(g, A, rev, ws, st, hs);
  return kind == RS_KIND_REFLECTOR ? launch_run<T, false, true>(g, A, rev, ws, st, hs)
                                   : launch_run<T, false, false>(g, A, rev, ws, st, hs);
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
  if (k > (int64_t)1 << 20) return fail(RS_EUNSUPPORTED, "more than 2^20 sequences");
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
                    int kind, void* ws, size_t bytes, void* stream, bool fast_only = false) {
  Geometry g;
  const int dtype = sizeof(T) == 8 ? RS_DTYPE_F64 : RS_DTYPE_F32;
  rs_status rc = validate(m, n, m > 1 ? m : 1, ldcs, k, side, order, kind, dtype, true, &g);
  if (rc != RS_OK) return rc;
  if (!C || !S) return fail(RS_EINVAL, "null pointer");
  rc = check_workspace(g, ws, bytes);
  if (rc != RS_OK) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int rev = order == RS_ORDER_REVERSE;
  // fast_only: the per-call fast path's pack (the scaled form unless it is disabled)
  const bool scaled = !fast_only || !scaled_disabled();
  return kind == RS_KIND_REFLECTOR ? launch_pack<T, true>(g, C, S, ldcs, rev, ws, st, scaled, fast_only)
                                   : launch_pack<T, false>(g, C, S, ldcs, rev, ws, st, scaled, fast_only);
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
    cudaError_t e = pool_alloc(&ws, need, st);
    if (e != cudaSuccess) return fail(RS_ENOMEM, std::string("workspace allocation: ") + cudaGetErrorString(e));
    owned = true;
  } else if (ws_bytes < need) {
    return fail(RS_ENOMEM, "workspace smaller than rs_workspace_bytes()");
  } else if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) {
    return fail(RS_EINVAL, "workspace must be 256-byte aligned");
  }
  const bool scaled = !strict && !scaled_disabled();
  rs_status rc = kind == RS_KIND_REFLECTOR ? launch_pack<T, true>(g, C, S, ldcs, rev, ws, st, scaled, true)
                                           : launch_pack<T, false>(g, C, S, ldcs, rev, ws, st, scaled, true);
  if (rc == RS_OK) rc = run_dispatch<T>(g, A, rev, kind, strict, ws, st);
  if (owned) {
    cudaError_t e = cudaFreeAsync(ws, st);
    if (rc == RS_OK && e != cudaSuccess) return fail(RS_ECUDA, std::string("cudaFreeAsync: ") + cudaGetErrorString(e));
  }
  return rc;
}

// ------------------------------------------------------------------------------------
// host-buffer entry point: A, C, S in host memory (pinned for full PCIe/C2C speed).
// C/S go first and are packed; A then streams in wave-column chunks on one copy stream
// while the pipeline kernel runs (its sweep-0 units wait for each chunk's arrival
// counter, written by a stream memory op after the copy), and every chunk streams back
// on a second copy stream as soon as all tiles' final units have released it (device
// counter awaited by a stream wait-value op). Copy-in, compute and copy-out overlap.
// ------------------------------------------------------------------------------------
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct StreamOps {
  PFN_writeValue32 write = nullptr;
  PFN_waitValue32 wait = nullptr;
  bool ok = false;
};

const StreamOps& stream_ops() {
  static StreamOps ops = [] {
    StreamOps o;
    void* fw = nullptr;
    void* fv = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    // the v2 stream memory ops (CUDA >= 12.0 ABI) are always available
    if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &fw, 12000, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &fv, 12000, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
      o.write = reinterpret_cast<PFN_writeValue32>(fw);
      o.wait = reinterpret_cast<PFN_waitValue32>(fv);
      o.ok = true;
    }
    return o;
  }();
  return ops;
}

// 2-D copy that degrades to a linear copy when both pitches equal the width (the copy
// engines run linear copies at full link speed; strided ones are slower)
cudaError_t copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                   cudaMemcpyKind kind, cudaStream_t st) {
  if (dpitch == width && spitch == width) return cudaMemcpyAsync(dst, src, width * height, kind, st);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, st);
}

// copy wave columns [v0, v1) of A between host (lda) and device (dense, ld = m)
template <typename T>
cudaError_t copy_wave_chunk(T* dev, T* host, const Geometry& g, int64_t m, int64_t lda, int rev, long long v0,
                            long long v1, cudaMemcpyKind kind, cudaStream_t st) {
  const long long p0 = rev ? g.len - v1 : v0;  // physical first column (right) / row (left)
  const long long cnt = v1 - v0;
  const bool left = g.os != 1;  // owners are columns
  T* dptr;
  T* hptr;
  size_t width, height;
  if (!left) {
    dptr = dev + p0 * m;
    hptr = host + p0 * lda;
    width = (size_t)m * sizeof(T);
    height = (size_t)cnt;
  } else {
    dptr = dev + p0;
    hptr = host + p0;
    width = (size_t)cnt * sizeof(T);
    height = (size_t)g.owners;
  }
  if (kind == cudaMemcpyHostToDevice)
    return copy2d(dptr, (size_t)m * sizeof(T), hptr, (size_t)lda * sizeof(T), width, height, kind, st);
  return copy2d(hptr, (size_t)lda * sizeof(T), dptr, (size_t)m * sizeof(T), width, height, kind, st);
}

constexpr int kMaxHostChunks = 64;
constexpr int kCopyLanes = 2;  // streams per direction (copies of a lane run on their own engine)
struct HostCtx {
  bool ready = false;
  cudaStream_t cin[kCopyLanes] = {}, cout[kCopyLanes] = {};
  cudaEvent_t e0 = nullptr, ecs = nullptr, eend[kCopyLanes] = {}, ejoin[kCopyLanes] = {};
  cudaEvent_t ein[kMaxHostChunks] = {};  // group i's arrival count is written
  uint32_t* ctl = nullptr;  // arrival / release counters (cudaMalloc: stream memory ops
                            // reject stream-ordered pool addresses)
};
constexpr int kMaxDevices = 64;

// One context per (host thread, device): calls alternating between devices reuse their
// own streams, events and counters instead of recreating (and leaking) them.
rs_status host_ctx(int dev, HostCtx** out) {
  static thread_local HostCtx ctxs[kMaxDevices];
  if (dev < 0 || dev >= kMaxDevices) return fail(RS_EUNSUPPORTED, "device ordinal >= 64");
  HostCtx& ctx = ctxs[dev];
  if (!ctx.ready) {
    bool okc = cudaEventCreateWithFlags(&ctx.e0, cudaEventDisableTiming) == cudaSuccess &&
               cudaEventCreateWithFlags(&ctx.ecs, cudaEventDisableTiming) == cudaSuccess &&
               cudaMalloc(reinterpret_cast<void**>(&ctx.ctl), (kMaxHostChunks + 1) * sizeof(uint32_t)) == cudaSuccess;
    for (int l = 0; l < kCopyLanes && okc; ++l)
      okc = cudaStreamCreateWithFlags(&ctx.cin[l], cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&ctx.cout[l], cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&ctx.eend[l], cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ctx.ejoin[l], cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < kMaxHostChunks && okc; ++i)
      okc = cudaEventCreateWithFlags(&ctx.ein[i], cudaEventDisableTiming) == cudaSuccess;
    if (!okc) return fail(RS_ECUDA, "stream/event/counter creation failed");
    ctx.ready = true;
  }
  *out = &ctx;
  return RS_OK;
}

template <typename T>
rs_status apply_host_impl(T* A, int64_t m, int64_t n, int64_t lda, const T* C, const T* S, int64_t ldcs, int64_t k,
                          int side, int order, int kind, int strict, void* stream) {
  const int dtype = sizeof(T) == 8 ? RS_DTYPE_F64 : RS_DTYPE_F32;
  Geometry gh;
  rs_status rc = validate(m, n, lda, ldcs, k, side, order, kind, dtype, true, &gh);
  if (rc != RS_OK) return rc;
  if (gh.owners == 0) return RS_OK;
  if (!A || !C || !S) return fail(RS_EINVAL, "null pointer");
  const StreamOps& ops = stream_ops();
  if (!ops.ok) return fail(RS_EUNSUPPORTED, "stream memory operations unavailable");
  Geometry g;  // device copy of A is dense: ld = m
  make_geometry(m, n, m > 1 ? m : 1, k, side, kind, dtype, &g);
  g.streaming = true;
  const int rev = order == RS_ORDER_REVERSE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  cudaGetDevice(&dev);
  HostCtx* ctxp = nullptr;
  rc = host_ctx(dev, &ctxp);
  if (rc != RS_OK) return rc;
  HostCtx& ctx = *ctxp;
  // wave-column chunks: ~64 per call, at least 16 columns each
  // Fine chunks (kernel-side arrival/release granularity) copied in groups that ramp up
  // and down (1, 1, 2, 4, G, ..., G, 4, 2, 1, 1 fine chunks): a small first group lets
  // the kernel start early, a small last group keeps the copy-out tail short, and the
  // large middle groups keep the copy engines at full speed.
  int nchunks_target = 64;
  if (const char* ev = getenv("RS_HOST_CHUNKS")) {
    const int v = atoi(ev);
    if (v >= 1 && v <= kMaxHostChunks) nchunks_target = v;
  }
  // groups of 2 fine chunks (~4 MB at config 2): measured best at config 2 (3.6 ms per call
  // against 4.1 ms with groups of 4 over 32 chunks): the copy-out stream starts earlier
  // and the two copy directions share the link more evenly
  int gmax = 2;
  if (const char* ev = getenv("RS_HOST_GROUP")) {
    const int v = atoi(ev);
    if (v >= 1) gmax = v;
  }
  int cw = (int)((g.len + nchunks_target - 1) / nchunks_target);
  if (cw < 16) cw = 16;
  const int ncw = (int)((g.len + cw - 1) / cw);
  int gb[kMaxHostChunks + 1];
  int ngroups = 0;
  {
    static const int ramp[] = {1, 1, 2, 4};
    int head[8], nh = 0, tailv[8], nt = 0, left = ncw;
    for (int r : ramp) {
      const int s = r < gmax ? r : gmax;
      if (left >= 2 * s) {
        head[nh++] = s;
        tailv[nt++] = s;
        left -= 2 * s;
      }
    }
    gb[0] = 0;
    int pos = 0;
    for (int i = 0; i < nh; ++i) gb[++ngroups] = (pos += head[i]);
    while (left > 0) {
      const int s = left < gmax ? left : gmax;
      gb[++ngroups] = (pos += s);
      left -= s;
    }
    for (int i = nt - 1; i >= 0; --i) gb[++ngroups] = (pos += tailv[i]);
  }
  const size_t abytes = (size_t)m * n * sizeof(T);
  const size_t csbytes = (size_t)(g.len - 1) * k * sizeof(T);
  const size_t wsbytes = g.coef_bytes + g.flag_bytes;
  const size_t ctlbytes = (size_t)(ncw + 1) * sizeof(uint32_t);
  unsigned char* mem = nullptr;
  const size_t off_c = align_up(abytes, 256), off_s = off_c + align_up(csbytes, 256);
  const size_t off_ws = off_s + align_up(csbytes, 256), off_ctl = off_ws + align_up(wsbytes, 256);  // = total
  cudaError_t e = pool_alloc(reinterpret_cast<void**>(&mem), off_ctl, st);
  if (e != cudaSuccess) return fail(RS_ENOMEM, std::string("device buffers: ") + cudaGetErrorString(e));
  T* dA = reinterpret_cast<T*>(mem);
  T* dC = reinterpret_cast<T*>(mem + off_c);
  T* dS = reinterpret_cast<T*>(mem + off_s);
  void* ws = mem + off_ws;
  uint32_t* ctl = ctx.ctl;  // [0] arrived, [1..ncw] done
  HostStream hs;
  hs.arrived = ctl;
  hs.done = ctl + 1;
  hs.cw = cw;
  hs.ncw = ncw;
  auto ck = [&](cudaError_t x, const char* what) -> bool {
    if (x != cudaSuccess && e == cudaSuccess) {
      e = x;
      g_err = std::string(what) + ": " + cudaGetErrorString(x);
    }
    return x == cudaSuccess;
  };
  e = cudaSuccess;
  // developer timeline (RS_HOST_DEBUG=1): events on every stream, printed to stderr
  const bool dbg = getenv("RS_HOST_DEBUG") != nullptr;
  cudaEvent_t dev_ev[3 * kMaxHostChunks + 8];
  int nev = 0;
  const char* ev_name[3 * kMaxHostChunks + 8];
  auto mark = [&](cudaStream_t s, const char* name) {
    if (!dbg || nev >= 3 * kMaxHostChunks + 8) return;
    cudaEventCreate(&dev_ev[nev]);
    cudaEventRecord(dev_ev[nev], s);
    ev_name[nev++] = name;
  };
  mark(st, "start");
  ck(cudaMemsetAsync(ctl, 0, ctlbytes, st), "memset");
  ck(cudaEventRecord(ctx.e0, st), "event");
  // copy-in stream: C, S, then A chunk by chunk, each followed by its arrival count
  int lanes = kCopyLanes;
  if (const char* ev = getenv("RS_HOST_LANES")) {
    const int v = atoi(ev);
    if (v >= 1 && v <= kCopyLanes) lanes = v;
  }
  for (int l = 0; l < lanes; ++l) ck(cudaStreamWaitEvent(ctx.cin[l], ctx.e0, 0), "wait");
  const size_t lc = (size_t)(g.len - 1);
  ck(copy2d(dC, lc * sizeof(T), C, (size_t)ldcs * sizeof(T), lc * sizeof(T), (size_t)k, cudaMemcpyHostToDevice,
            ctx.cin[0]), "C copy");
  ck(copy2d(dS, lc * sizeof(T), S, (size_t)ldcs * sizeof(T), lc * sizeof(T), (size_t)k, cudaMemcpyHostToDevice,
            ctx.cin[0]), "S copy");
  ck(cudaEventRecord(ctx.ecs, ctx.cin[0]), "event");
  mark(ctx.cin[0], "cs_in");
  static const char* kInNames[] = {"in0", "in1", "in2", "in3", "in4", "in5", "in6", "in7", "in8", "in9"};
  static const char* kOutNames[] = {"out0", "out1", "out2", "out3", "out4", "out5", "out6", "out7", "out8", "out9"};
  // groups alternate over the copy lanes; a group's arrival count is written only after
  // the previous group's (event chain), so the counter only grows
  for (int gi = 0; gi < ngroups && e == cudaSuccess; ++gi) {
    cudaStream_t cs_ = ctx.cin[gi % lanes];
    if (gi < 10) mark(cs_, kInNames[gi]);
    const long long v0 = (long long)gb[gi] * cw;
    const long long v1 = (long long)gb[gi + 1] * cw < g.len ? (long long)gb[gi + 1] * cw : g.len;
    ck(copy_wave_chunk<T>(dA, A, g, m, lda, rev, v0, v1, cudaMemcpyHostToDevice, cs_), "A copy-in");
    if (gi > 0 && lanes > 1) ck(cudaStreamWaitEvent(cs_, ctx.ein[gi - 1], 0), "wait");
    const CUresult r = ops.write(reinterpret_cast<CUstream>(cs_), reinterpret_cast<CUdeviceptr>(ctl),
                                 (cuuint32_t)gb[gi + 1], 0);
    ck(cudaEventRecord(ctx.ein[gi], cs_), "event");
    if (r != CUDA_SUCCESS) {
      ck(cudaErrorUnknown, "cuStreamWriteValue32");
      g_err += " (CUresult " + std::to_string((int)r) + ")";
    }
  }
  mark(ctx.cin[(ngroups - 1) % lanes], "a_in_done");
  // compute stream: pack once C/S are in, then the streaming pipeline kernel
  ck(cudaStreamWaitEvent(st, ctx.ecs, 0), "wait");
  mark(st, "pack_start");
  if (e == cudaSuccess) {
    const bool scaled = !strict && !scaled_disabled();
    rc = kind == RS_KIND_REFLECTOR ? launch_pack<T, true>(g, dC, dS, (long long)lc, rev, ws, st, scaled, true)
                                   : launch_pack<T, false>(g, dC, dS, (long long)lc, rev, ws, st, scaled, true);
    mark(st, "kernel_start");
    if (rc == RS_OK) rc = run_dispatch<T>(g, dA, rev, kind, strict, ws, st, &hs);
    mark(st, "kernel_end");
  }
  // copy-out stream: chunk i leaves once every tile's final unit has released it
  for (int l = 0; l < lanes; ++l) ck(cudaStreamWaitEvent(ctx.cout[l], ctx.e0, 0), "wait");
  for (int gi = 0; gi < ngroups && e == cudaSuccess && rc == RS_OK; ++gi) {
    // final units release chunks in order, so the group's last chunk implies the rest
    cudaStream_t co_ = ctx.cout[gi % lanes];
    const CUresult r = ops.wait(reinterpret_cast<CUstream>(co_),
                                reinterpret_cast<CUdeviceptr>(ctl + gb[gi + 1]), (cuuint32_t)g.tiles,
                                CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) {
      ck(cudaErrorUnknown, "cuStreamWaitValue32");
      g_err += " (CUresult " + std::to_string((int)r) + ")";
    }
    const long long v0 = (long long)gb[gi] * cw;
    const long long v1 = (long long)gb[gi + 1] * cw < g.len ? (long long)gb[gi + 1] * cw : g.len;
    if (gi < 10) mark(co_, kOutNames[gi]);
    ck(copy_wave_chunk<T>(dA, A, g, m, lda, rev, v0, v1, cudaMemcpyDeviceToHost, co_), "A copy-out");
  }
  mark(ctx.cout[(ngroups - 1) % lanes], "out_done");
  // join every copy lane (in and out) into st on every path, success or error: no H2D
  // copy or arrival write into `mem` / ctx.ctl may still be pending when `mem` returns to
  // the pool or the next call resets the counters
  for (int l = 0; l < lanes; ++l) {
    cudaEventRecord(ctx.ejoin[l], ctx.cin[l]);
    cudaStreamWaitEvent(st, ctx.ejoin[l], 0);
    cudaEventRecord(ctx.eend[l], ctx.cout[l]);
    cudaStreamWaitEvent(st, ctx.eend[l], 0);
  }
  cudaFreeAsync(mem, st);
  cudaError_t es = cudaStreamSynchronize(st);
  if (dbg) {
    cudaDeviceSynchronize();
    for (int i = 0; i < nev; ++i) {
      float ms = 0;
      const cudaError_t ee = cudaEventElapsedTime(&ms, dev_ev[0], dev_ev[i]);
      fprintf(stderr, "[rs_apply_host] %-16s %8.3f ms %s\n", ev_name[i], ms, ee == cudaSuccess ? "" : cudaGetErrorString(ee));
    }
    for (int i = 0; i < nev; ++i) cudaEventDestroy(dev_ev[i]);
  }
  if (rc != RS_OK) return rc;
  if (e != cudaSuccess) return RS_ECUDA;
  if (es != cudaSuccess) return fail(RS_ECUDA, std::string("rs_apply_host: ") + cudaGetErrorString(es));
  return RS_OK;
}

// micro-kernel API launcher (kernel_wave_apply, kernels.py:335-371)
template <typename T, bool STRICT, bool REFL, int KR>
cudaError_t launch_wave_kr(T* P, long long m_r, long long ld, const T* ct, const T* st, long long n_waves,
                           long long col0, cudaStream_t s) {
  const size_t smem = (size_t)2 * kWaveChunkBlocks * (KR + 1) * KR * sizeof(T);
  const unsigned blocks = (unsigned)((m_r + 127) / 128);
  rs_wave_kernel<T, KR, STRICT, REFL><<<blocks, 128, smem, s>>>(P, m_r, ld, ct, st, n_waves, col0);
  return cudaGetLastError();
}
template <typename T, bool STRICT, bool REFL>
cudaError_t launch_wave(T* P, long long m_r, long long ld, const T* ct, const T* st, long long n_waves, int k_r,
                        long long col0, cudaStream_t s) {
  switch (k_r) {
    case 1: return launch_wave_kr<T, STRICT, REFL, 1>(P, m_r, ld, ct, st, n_waves, col0, s);
    case 2: return launch_wave_kr<T, STRICT, REFL, 2>(P, m_r, ld, ct, st, n_waves, col0, s);
    case 3: return launch_wave_kr<T, STRICT, REFL, 3>(P, m_r, ld, ct, st, n_waves, col0, s);
    case 4: return launch_wave_kr<T, STRICT, REFL, 4>(P, m_r, ld, ct, st, n_waves, col0, s);
    case 5: return launch_wave_kr<T, STRICT, REFL, 5>(P, m_r, ld, ct, st, n_waves, col0, s);
    case 6: return launch_wave_kr<T, STRICT, REFL, 6>(P, m_r, ld, ct, st, n_waves, col0, s);
    case 7: return launch_wave_kr<T, STRICT, REFL, 7>(P, m_r, ld, ct, st, n_waves, col0, s);
    case 8: return launch_wave_kr<T, STRICT, REFL, 8>(P, m_r, ld, ct, st, n_waves, col0, s);
    default: {
      const unsigned blocks = (unsigned)((m_r + 127) / 128);
      rs_wave_kernel_wide<T, STRICT, REFL><<<blocks, 128, 0, s>>>(P, m_r, ld, ct, st, n_waves, k_r, col0);
      return cudaGetLastError();
    }
  }
}
template <typename T>
rs_status wave_impl(T* P, int64_t m_r, int64_t n_cols, int64_t ld, const T* ct, const T* st, int64_t n_waves,
                    int64_t k_r, int64_t col0, int kind, int strict, void* stream) {
  if (kind != RS_KIND_ROTATION && kind != RS_KIND_REFLECTOR)
    return fail(RS_EINVAL, "kind must be 0 (rotation) or 1 (reflector)");
  if (m_r < 0 || n_cols < 0 || n_waves < 0 || col0 < 0) return fail(RS_EINVAL, "sizes must be non-negative");
  if (k_r < 1) return fail(RS_EINVAL, "kernel shape must be positive (k_r >= 1)");
  if (k_r > (1 << 20)) return fail(RS_EUNSUPPORTED, "k_r larger than 2^20");
  if (ld < (m_r > 1 ? m_r : 1)) return fail(RS_EINVAL, "ld must be >= max(1, m_r)");
  if (n_cols - col0 < n_waves + k_r)
    return fail(RS_EINVAL, "panel has " + std::to_string(n_cols - col0) + " usable columns, need " +
                               std::to_string(n_waves + k_r) + " for " + std::to_string(n_waves) + " waves of " +
                               std::to_string(k_r));
  if (m_r == 0 || n_waves == 0) return RS_OK;
  if (!P || !ct || !st) return fail(RS_EINVAL, "null pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (strict)
    e = kind == RS_KIND_REFLECTOR ? launch_wave<T, true, true>(P, m_r, ld, ct, st, n_waves, (int)k_r, col0, s)
                                  : launch_wave<T, true, false>(P, m_r, ld, ct, st, n_waves, (int)k_r, col0, s);
  else
    e = kind == RS_KIND_REFLECTOR ? launch_wave<T, false, true>(P, m_r, ld, ct, st, n_waves, (int)k_r, col0, s)
                                  : launch_wave<T, false, false>(P, m_r, ld, ct, st, n_waves, (int)k_r, col0, s);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (e != cudaSuccess) return fail(RS_ECUDA, std::string("wave kernel launch: ") + cudaGetErrorString(e));
  return RS_OK;
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
  rs_status rc = plan_launch(g, dtype == RS_DTYPE_F64 ? 8 : 4, &lp);
  if (rc != RS_OK) return rc;
  if (grid_ctas) *grid_ctas = lp.grid;
  if (warps_per_cta) *warps_per_cta = lp.nw;
  if (units) *units = lp.units;
  if (band_width) *band_width = g.kw;
  if (rows_per_tile) *rows_per_tile = tile_owners(dtype == RS_DTYPE_F64 ? 8 : 4);
  if (smem_bytes) *smem_bytes = lp.smem;
  return RS_OK;
}

rs_status rs_tile_shape(int dtype, int side, int* window_sweeps, int* rows_per_thread, int* ring_chunks,
                        int* small_cta_warps, int* max_warps) {
  g_err.clear();
  if (dtype != RS_DTYPE_F64 && dtype != RS_DTYPE_F32) return fail(RS_EINVAL, "bad dtype");
  if (side != RS_SIDE_LEFT && side != RS_SIDE_RIGHT) return fail(RS_EINVAL, "bad side");
  const size_t tsz = dtype == RS_DTYPE_F64 ? 8 : 4;
  const bool left = side == RS_SIDE_LEFT;
  if (window_sweeps) *window_sweeps = kK;
  if (rows_per_thread) *rows_per_thread = rows_for(tsz);
  if (ring_chunks) *ring_chunks = stages_for(tsz);
  if (small_cta_warps) *small_cta_warps = (tsz == 8 && !left) ? kSmallCtaWarps : 0;
  if (max_warps) *max_warps = max_warps_for(tsz, left, kK);
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
rs_status rs_pack_fast_f64(const double* C, const double* S, int64_t ldcs, int64_t m, int64_t n, int64_t k,
                           int side, int order, int kind, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  return pack_impl<double>(C, S, ldcs, m, n, k, side, order, kind, workspace, workspace_bytes, stream, true);
}
rs_status rs_pack_fast_f32(const float* C, const float* S, int64_t ldcs, int64_t m, int64_t n, int64_t k,
                           int side, int order, int kind, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  return pack_impl<float>(C, S, ldcs, m, n, k, side, order, kind, workspace, workspace_bytes, stream, true);
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

rs_status rs_packed_form(const void* workspace, size_t workspace_bytes, int64_t m, int64_t n, int64_t k,
                         int side, int kind, int dtype, int64_t* scaled_units, int64_t* total_units, void* stream) {
  g_err.clear();
  if (!scaled_units || !total_units) return fail(RS_EINVAL, "null pointer");
  if (dtype != RS_DTYPE_F64 && dtype != RS_DTYPE_F32) return fail(RS_EINVAL, "dtype must be 0 (f64) or 1 (f32)");
  Geometry g;
  rs_status rc = validate(m, n, m > 1 ? m : 1, 0, k, side, RS_ORDER_FORWARD, kind, dtype, false, &g);
  if (rc != RS_OK) return rc;
  rc = check_workspace(g, const_cast<void*>(workspace), workspace_bytes);
  if (rc != RS_OK) return rc;
  LaunchPlan lp;
  rc = plan_launch(g, dtype == RS_DTYPE_F64 ? 8 : 4, &lp);
  if (rc != RS_OK) return rc;
  const int nw = 2 * (lp.ua + 1);
  uint32_t flags[2 * (kK + 1) + 2];
  uint32_t* host = nw <= (int)(sizeof(flags) / sizeof(flags[0])) ? flags : (uint32_t*)malloc(nw * sizeof(uint32_t));
  if (!host) return fail(RS_ENOMEM, "host buffer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const unsigned char* base = reinterpret_cast<const unsigned char*>(workspace) + g.coef_bytes + g.flags_only;
  cudaError_t e = cudaMemcpyAsync(host, base, nw * sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    if (host != flags) free(host);
    return fail(RS_ECUDA, std::string("rs_packed_form: ") + cudaGetErrorString(e));
  }
  // part 1: the first t1 tiles, ua+1 units each; part 0: the others, ua units each
  long long scaled = 0;
  const bool off = scaled_disabled();
  for (int part = 0; part < 2; ++part) {
    const long long tiles = part ? lp.t1 : g.tiles - lp.t1;
    const int ut = lp.ua + part;
    for (int i = 0; i < ut && tiles > 0; ++i)
      if (!off && host[part * (lp.ua + 1) + i] == 0u) scaled += tiles;
  }
  if (host != flags) free(host);
  *scaled_units = scaled;
  *total_units = lp.units;
  return RS_OK;
}

rs_status rs_apply_host_f64(double* A, int64_t m, int64_t n, int64_t lda, const double* C, const double* S,
                            int64_t ldcs, int64_t k, int side, int order, int kind, int strict, void* stream) {
  g_err.clear();
  return apply_host_impl<double>(A, m, n, lda, C, S, ldcs, k, side, order, kind, strict, stream);
}
rs_status rs_apply_host_f32(float* A, int64_t m, int64_t n, int64_t lda, const float* C, const float* S,
                            int64_t ldcs, int64_t k, int side, int order, int kind, int strict, void* stream) {
  g_err.clear();
  return apply_host_impl<float>(A, m, n, lda, C, S, ldcs, k, side, order, kind, strict, stream);
}

rs_status rs_wave_apply_f64(double* panel, int64_t m_r, int64_t n_cols, int64_t ld, const double* ct,
                            const double* st, int64_t n_waves, int64_t k_r, int64_t col0, int kind, int strict,
                            void* stream) {
  g_err.clear();
  return wave_impl<double>(panel, m_r, n_cols, ld, ct, st, n_waves, k_r, col0, kind, strict, stream);
}
rs_status rs_wave_apply_f32(float* panel, int64_t m_r, int64_t n_cols, int64_t ld, const float* ct,
                            const float* st, int64_t n_waves, int64_t k_r, int64_t col0, int kind, int strict,
                            void* stream) {
  g_err.clear();
  return wave_impl<float>(panel, m_r, n_cols, ld, ct, st, n_waves, k_r, col0, kind, strict, stream);
}

size_t rs_dmma_workspace_bytes(int64_t m, int64_t n, int64_t k) { return dmma_workspace(m, n, k); }

rs_status rs_apply_dmma_f64(double* A, int64_t m, int64_t n, int64_t lda, const double* C, const double* S,
                            int64_t ldcs, int64_t k, int order, int kind, void* workspace, size_t workspace_bytes,
                            void* stream) {
  g_err.clear();
  if (order != RS_ORDER_FORWARD && order != RS_ORDER_REVERSE)
    return fail(RS_EINVAL, "order must be 0 (forward) or 1 (reverse)");
  if (kind != RS_KIND_ROTATION && kind != RS_KIND_REFLECTOR)
    return fail(RS_EINVAL, "kind must be 0 (rotation) or 1 (reflector)");
  if (m < 0 || n < 0) return fail(RS_EINVAL, "matrix dimensions must be non-negative");
  if (n < 2) return fail(RS_EINVAL, "matrix needs at least 2 columns");
  if (n > ((int64_t)1 << 26)) return fail(RS_EUNSUPPORTED, "rotated dimension longer than 2^26");
  if (k < 1) return fail(RS_EINVAL, "need k >= 1 sequences");
  if (k > ((int64_t)1 << 20)) return fail(RS_EUNSUPPORTED, "more than 2^20 sequences");
  if (lda < (m > 1 ? m : 1)) return fail(RS_EINVAL, "lda must be >= max(1, m) (column-major)");
  if (ldcs < n - 1) return fail(RS_EINVAL, "ldcs must be >= len - 1");
  if (m == 0) return RS_OK;
  if (!A || !C || !S) return fail(RS_EINVAL, "null pointer");
  const size_t need = dmma_workspace(m, n, k);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  void* ws = workspace;
  bool owned = false;
  if (ws == nullptr) {
    cudaError_t e = pool_alloc(&ws, need, st);
    if (e != cudaSuccess) return fail(RS_ENOMEM, std::string("workspace allocation: ") + cudaGetErrorString(e));
    owned = true;
  } else if (workspace_bytes < need) {
    return fail(RS_ENOMEM, "workspace smaller than rs_dmma_workspace_bytes()");
  } else if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) {
    return fail(RS_EINVAL, "workspace must be 256-byte aligned");
  }
  const int launched = dmma_run(A, m, n, lda, C, S, ldcs, k, order == RS_ORDER_REVERSE,
                                kind == RS_KIND_REFLECTOR, ws, st);
  if (launched > 0) g_launches.fetch_add(launched, std::memory_order_relaxed);
  if (owned) cudaFreeAsync(ws, st);
  if (launched < 0) return fail(RS_ECUDA, std::string("dmma launch: ") + cudaGetErrorString(cudaGetLastError()));
  return RS_OK;
}

rs_status rs_debug_set_trace(void* device_ptr) {
  g_err.clear();
#ifndef RS_TRACE
  (void)device_ptr;
  return fail(RS_EUNSUPPORTED, "library built without -DRS_TRACE");
#endif
  g_trace_buf = reinterpret_cast<unsigned long long*>(device_ptr);
  return RS_OK;
}

}  // extern "C"
