// dmma_variant.cu — the accumulate-and-apply variant on the FP64 tensor cores (DMMA).
//
// The paper's rs_gemm idea and the reference's explicit-Q oracle
// (accumulate_q, oracle.py:102-109), done per block of the wavefront: the k sweeps are
// cut into passes of KB = 32 sweeps; inside a pass the waves t = j + l (lane l = sweep
// p0 + l rotates columns (t - l, t - l + 1), the reference's wavefront order,
// core.py:152-172) are cut into windows of NB = 32 waves. All rotations of window w touch
// only the W = NB + KB = 64 columns c0(w) = w*NB - KB + 1 .. c0(w) + 63, so their product is
// a 64 x 64 matrix Q_w, and the pass is
//     A[:, cols(w)] <- A[:, cols(w)] * Q_w        for w = 0, 1, ... in order
// (windows overlap by KB columns; wave order is dependency-legal, so the result equals
// the plain loop up to rounding). Q_w is built once per call (rs_dmma_q_kernel: 64 threads,
// thread i carries row i of Q through the window's rotations in the reference's order) and
// applied with mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) by rs_dmma_apply_kernel: a CTA owns 32
// rows of A and streams the windows, keeping the 64 window columns in a 96-column shared
// ring (the next 32 columns prefetched by cp.async while the current window multiplies),
// Q_w double-buffered by a TMA bulk copy, and 8x8 tiles of Q_w that are structurally zero
// (the parallelogram's corners: 12 of 64 tiles) skipped.
//
// Counted flops are the reference's 6*m*(n-1)*k; the tensor cores execute
// 2*32*64*64*(52/64) per 32 rows and window, 1.08x that. Fast-mode arithmetic: the result
// is within the BASELINE tolerance of the reference, not bit-identical (products of
// rotations are reassociated). Right side, both orders, both kinds, fp64.

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "rotseq_b200.h"
#include "rotseq_device.cuh"

namespace rsk {

constexpr int kDNB = 32;               // waves per window
constexpr int kDKB = 32;               // sweeps per pass
constexpr int kDW = kDNB + kDKB;       // window columns (64)
constexpr int kDRows = 32;             // rows of A per CTA
constexpr int kDColStride = kDRows + 4;  // shared column stride (doubles): conflict-free A fragments
constexpr int kDRing = 3 * 32;         // shared column ring (3 groups of 32)
constexpr int kDQ = kDW * kDW;         // doubles per Q_w

__host__ __device__ inline int dmma_windows(int n) { return (n + kDKB - 2 + kDNB - 1) / kDNB; }

// Q_w for (pass, window) = (blockIdx.y, blockIdx.x). Thread i keeps row i of Q in shared
// memory and applies the window's rotations in wave order, lanes ascending (column
// operations Q <- Q * G, as accumulate_q does). Output in DMMA B-fragment order:
// Qf[(ks * 8 + nt) * 32 + lane] = Q[ks*4 + lane%4][nt*8 + lane/4]; plus a 64-bit mask of the
// nonzero 8x8 tiles (bit kt*8 + nt).
template <bool REFL>
__global__ void __launch_bounds__(kDW) rs_dmma_q_kernel(double* __restrict__ qout, unsigned long long* __restrict__ masks,
                                                        const double* __restrict__ C, const double* __restrict__ S,
                                                        long long ldcs, int n, int k, int rev) {
  __shared__ double q[kDW][kDW + 1];
  __shared__ unsigned long long tile_bits[kDW];
  const int i = threadIdx.x;
  const int w = blockIdx.x, pass = blockIdx.y;
  const int p0 = pass * kDKB;
  const int lanes = k - p0 < kDKB ? k - p0 : kDKB;
#pragma unroll 8
  for (int c = 0; c < kDW; ++c) q[i][c] = c == i ? 1.0 : 0.0;
  const int c0 = w * kDNB - kDKB + 1;
  for (int t = w * kDNB; t < (w + 1) * kDNB; ++t) {
    for (int l = 0; l < lanes; ++l) {
      const int j = t - l;
      if (j < 0 || j > n - 2) continue;
      const long long jj = rev ? (long long)(n - 2 - j) : (long long)j;
      double c = __ldg(C + jj + (long long)(p0 + l) * ldcs);
      double s = __ldg(S + jj + (long long)(p0 + l) * ldcs);
      const int x = j - c0;
      const double qx = q[i][x], qy = q[i][x + 1];
      if constexpr (REFL) {
        if (rev) c = -c;
        const double w2 = s * (qx + qy);
        q[i][x] = fma(c - s, qx, w2);
        q[i][x + 1] = fma(-(c + s), qy, w2);
      } else {
        if (rev) s = -s;
        q[i][x] = fma(s, qy, c * qx);
        q[i][x + 1] = fma(c, qy, -s * qx);
      }
    }
  }
  // fragment-order store and the nonzero-tile mask
  double* const qw = qout + ((size_t)pass * gridDim.x + w) * kDQ;
  const int ks = i >> 2, lq = i & 3;
  unsigned long long bits = 0;
#pragma unroll 8
  for (int c = 0; c < kDW; ++c) {
    const double v = q[i][c];
    qw[(ks * 8 + (c >> 3)) * 32 + lq + 4 * (c & 7)] = v;
    if (v != 0.0) bits |= 1ull << ((i >> 3) * 8 + (c >> 3));
  }
  tile_bits[i] = bits;
  __syncthreads();
  if (i == 0) {
    unsigned long long m = 0;
    for (int r = 0; r < kDW; ++r) m |= tile_bits[r];
    masks[(size_t)pass * gridDim.x + w] = m;
  }
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// One pass over all windows for 32 rows of A (right side; A column-major, lda).
__global__ void __launch_bounds__(256, 1) rs_dmma_apply_kernel(double* __restrict__ A, long long m, long long lda,
                                                               int n, const double* __restrict__ qpass,
                                                               const unsigned long long* __restrict__ mpass,
                                                               int nwin) {
  extern __shared__ __align__(128) unsigned char dsm[];
  double* const qbuf = reinterpret_cast<double*>(dsm);                 // 2 x kDQ
  double* const ring = qbuf + 2 * kDQ;                                 // kDRing x kDColStride
  uint64_t* const qbar = reinterpret_cast<uint64_t*>(ring + kDRing * kDColStride);  // 2 mbarriers
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long r0 = (long long)blockIdx.x * kDRows;
  if (tid == 0) {
    mbar_init(&qbar[0], 1);
    mbar_init(&qbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // column c of A lives in ring slot ((c + KB - 1) mod 96); a group of 32 columns starts at
  // c0(w) + 32 g. Cooperative cp.async of group g (32 columns x 32 rows, one element per
  // copy: any lda; columns or rows outside the matrix are zero-filled).
  auto load_group = [&](int g) {
    const int cbase = g * 32 - kDKB + 1;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int idx = tid + it * 256;  // 1024 elements: column cl = idx / 32, row idx % 32
      const int cl = idx >> 5, rr = idx & 31;
      const int col = cbase + cl;
      const long long row = r0 + rr;
      const bool ok = col >= 0 && col < n && row < m;
      cp_async_elem(ring + ((g % 3) * 32 + cl) * kDColStride + rr, ok ? A + (long long)col * lda + row : A, ok);
    }
    cp_async_commit();
  };
  auto issue_q = [&](int w) {
    if (tid == 0 && w < nwin) {
      uint64_t* bar = &qbar[w & 1];
      // the buffer's previous readers were generic-proxy loads (window w - 2)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, kDQ * 8);
      bulk_g2s_nowait(qbuf + (w & 1) * kDQ, qpass + (size_t)w * kDQ, kDQ * 8, bar);
    }
  };
  // prologue: groups 0 and 1 (window 0), Q_0
  load_group(0);
  load_group(1);
  issue_q(0);
  const int nt = warp;  // this warp's 8 output columns of the window
  for (int w = 0; w < nwin; ++w) {
    // prefetch: the next window's new columns (group w + 2) and Q_{w+1}
    if (w + 1 < nwin) load_group(w + 2); else cp_async_commit();
    issue_q(w + 1);
    cp_async_wait_group<1>();  // groups w, w + 1 have landed (this thread's copies)
    __syncthreads();           // ... everyone's copies, and window w-1's carried outputs
    mbar_wait(&qbar[w & 1], (uint32_t)(w >> 1) & 1u);
    const double* const qs = qbuf + (w & 1) * kDQ;
    const unsigned long long mask = __ldg(mpass + w);
    double acc[4][2];
#pragma unroll
    for (int rt = 0; rt < 4; ++rt) acc[rt][0] = acc[rt][1] = 0.0;
    const int sbase = (w % 3) * 32;  // ring slot of the window's first column
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
      if (!((mask >> (kt * 8 + nt)) & 1ull)) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ks = kt * 2 + h;
        const double b = qs[(ks * 8 + nt) * 32 + lane];
        int slot = sbase + ks * 4 + (lane & 3);
        if (slot >= kDRing) slot -= kDRing;
        const double* xc = ring + slot * kDColStride + (lane >> 2);
#pragma unroll
        for (int rt = 0; rt < 4; ++rt) dmma884(acc[rt], xc[rt * 8], b);
      }
    }
    __syncthreads();  // all reads of groups w, w + 1 and of Q_w are done
    // outputs: columns 0..31 of the window are final for this pass (to A), 32..63 are
    // carried into the next window (group w + 1's slots, in place)
    const int ocol = nt * 8 + (lane & 3) * 2;  // window column of acc[.][0]
#pragma unroll
    for (int rt = 0; rt < 4; ++rt) {
      const int rr = rt * 8 + (lane >> 2);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int wc = ocol + e;
        if (nt < 4) {
          const int col = w * kDNB - kDKB + 1 + wc;
          const long long row = r0 + rr;
          if (col >= 0 && col < n && row < m) A[(long long)col * lda + row] = acc[rt][e];
        } else {
          int slot = sbase + wc;
          if (slot >= kDRing) slot -= kDRing;
          ring[slot * kDColStride + rr] = acc[rt][e];
        }
      }
    }
  }
  cp_async_wait_group<0>();
  __syncthreads();
  // the last window's carried columns (group nwin) are final too
  {
    const int g = nwin;
    for (int idx = tid; idx < 32 * kDRows; idx += 256) {
      const int cl = idx / kDRows, rr = idx % kDRows;
      const int col = g * 32 - kDKB + 1 + cl;
      const long long row = r0 + rr;
      if (col >= 0 && col < n && row < m) A[(long long)col * lda + row] = ring[((g % 3) * 32 + cl) * kDColStride + rr];
    }
  }
}

size_t dmma_workspace(int64_t m, int64_t n, int64_t k) {
  if (m < 0 || n < 2 || k < 1) return 0;
  const int64_t passes = (k + kDKB - 1) / kDKB;
  const int64_t nwin = dmma_windows((int)n);
  return (size_t)(passes * nwin) * (kDQ * sizeof(double) + sizeof(unsigned long long)) + 256;
}

// Launches the Q-build kernel and one apply kernel per pass on `st`; returns the number of
// kernels launched (negative: launch error, cudaGetLastError() tells which).
int dmma_run(double* A, int64_t m, int64_t n, int64_t lda, const double* C, const double* S, int64_t ldcs,
             int64_t k, int rev, int refl, void* workspace, cudaStream_t st) {
  const int passes = (int)((k + kDKB - 1) / kDKB);
  const int nwin = dmma_windows((int)n);
  double* q = reinterpret_cast<double*>(workspace);
  unsigned long long* masks = reinterpret_cast<unsigned long long*>(q + (size_t)passes * nwin * kDQ);
  dim3 qg((unsigned)nwin, (unsigned)passes);
  if (refl)
    rs_dmma_q_kernel<true><<<qg, kDW, 0, st>>>(q, masks, C, S, ldcs, (int)n, (int)k, rev);
  else
    rs_dmma_q_kernel<false><<<qg, kDW, 0, st>>>(q, masks, C, S, ldcs, (int)n, (int)k, rev);
  const size_t smem = (size_t)2 * kDQ * 8 + (size_t)kDRing * kDColStride * 8 + 2 * sizeof(uint64_t);
  static std::atomic<int> configured{0};
  if (!configured.load()) {
    if (cudaFuncSetAttribute(rs_dmma_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return -1;
    configured.store(1);
  }
  // reverse order: mirror the columns (base at the last column, negative stride)
  double* Ab = rev ? A + (long long)(n - 1) * lda : A;
  const long long ld = rev ? -lda : lda;
  const unsigned grid = (unsigned)((m + kDRows - 1) / kDRows);
  for (int p = 0; p < passes; ++p)
    rs_dmma_apply_kernel<<<grid, 256, smem, st>>>(Ab, m, ld, (int)n, q + (size_t)p * nwin * kDQ,
                                                  masks + (size_t)p * nwin, nwin);
  return cudaPeekAtLastError() == cudaSuccess ? passes + 1 : -1;
}

}  // namespace rsk
