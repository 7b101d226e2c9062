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
// rows of A and streams the windows, the 64 window columns in shared memory (32 carried
// from the previous window, 32 new ones prefetched by cp.async while the current window
// multiplies),
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
constexpr int kDQ = kDW * kDW;         // doubles per Q_w

__host__ __device__ inline int dmma_windows(int n) { return (n + kDKB - 2 + kDNB - 1) / kDNB; }

// Q_w for (pass, window) = (blockIdx.y, blockIdx.x). The window's coefficients (rotation
// pairs j in [c0, c0 + 62], the pass's lanes) are staged in shared memory first, then thread
// i keeps row i of Q in registers and applies the window's rotations in wave order, lanes
// ascending (column operations Q <- Q * G, as accumulate_q does). Output in DMMA
// B-fragment order: Qf[(ks * 8 + nt) * 32 + lane] = Q[ks*4 + lane%4][nt*8 + lane/4]; plus a
// 64-bit mask of the nonzero 8x8 tiles (bit kt*8 + nt).
constexpr int kDPairs = kDW - 1;  // rotation pairs a window can touch (63)
template <bool REFL>
__global__ void __launch_bounds__(kDW) rs_dmma_q_kernel(double* __restrict__ qout, unsigned long long* __restrict__ masks,
                                                        const double* __restrict__ C, const double* __restrict__ S,
                                                        long long ldcs, int n, int k, int rev) {
  extern __shared__ __align__(16) unsigned char qsm[];
  double2 (*cs)[kDPairs] = reinterpret_cast<double2 (*)[kDPairs]>(qsm);  // (c, s) of pair c0 + x, lane l
  __shared__ unsigned long long tile_bits[kDW];
  const int i = threadIdx.x;
  const int w = blockIdx.x, pass = blockIdx.y;
  const int p0 = pass * kDKB;
  const int lanes = k - p0 < kDKB ? k - p0 : kDKB;
  const int c0 = w * kDNB - kDKB + 1;
  // pairs outside the matrix and lanes past the pass are staged as identities (c, s) = (1, 0):
  // the rotation loop below then needs no predicates (an identity is exact)
  for (int e = i; e < kDKB * kDPairs; e += kDW) {
    const int l = e / kDPairs, x = e - l * kDPairs;
    const int j = c0 + x;
    double c = 1.0, s = 0.0;
    bool id = true;
    if (l < lanes && j >= 0 && j <= n - 2) {
      const long long jj = rev ? (long long)(n - 2 - j) : (long long)j;
      c = __ldg(C + jj + (long long)(p0 + l) * ldcs);
      s = __ldg(S + jj + (long long)(p0 + l) * ldcs);
      if (rev) {
        if constexpr (REFL) c = -c; else s = -s;
      }
      id = false;
    }
    if constexpr (REFL) {
      // a reflector is not an identity for any (c, s): mark skipped pairs with s = NaN
      if (id) s = __longlong_as_double(0x7ff8000000000001ll);
    }
    cs[l][x] = make_double2(c, s);
  }
  __syncthreads();
  // row i of Q in registers: column x of the window is q[x] (compile-time indices: the
  // wave and lane loops are fully unrolled, x = (t - 32 w) + 31 - l)
  double q[kDW];
#pragma unroll
  for (int c = 0; c < kDW; ++c) q[c] = c == i ? 1.0 : 0.0;
#pragma unroll
  for (int tt = 0; tt < kDNB; ++tt) {
#pragma unroll
    for (int l = 0; l < kDKB; ++l) {
      const int x = tt + kDKB - 1 - l;
      const double2 r = cs[l][x];
      const double qx = q[x], qy = q[x + 1];
      if constexpr (REFL) {
        if (r.y == r.y) {  // not a skipped pair (NaN marker)
          const double w2 = r.y * (qx + qy);
          q[x] = fma(r.x - r.y, qx, w2);
          q[x + 1] = fma(-(r.x + r.y), qy, w2);
        }
      } else {
        q[x] = fma(r.y, qy, r.x * qx);
        q[x + 1] = fma(r.x, qy, -r.y * qx);
      }
    }
  }
  // fragment-order store and the nonzero-tile mask
  double* const qw = qout + ((size_t)pass * gridDim.x + w) * kDQ;
  const int ks = i >> 2, lq = i & 3;
  unsigned long long bits = 0;
#pragma unroll
  for (int c = 0; c < kDW; ++c) {
    qw[(ks * 8 + (c >> 3)) * 32 + lq + 4 * (c & 7)] = q[c];
    if (q[c] != 0.0) bits |= 1ull << ((i >> 3) * 8 + (c >> 3));
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

// One pass over all windows for 32 rows of A (right side; A column-major, lda; a negative
// lda walks the columns backwards for reverse order). Window w's 64 columns are its 32
// carried columns (cbuf[(w+1)&1]: window w-1's outputs 32..63, already rotated by the
// earlier windows of this pass) followed by 32 new columns from A (nbuf[w&1], prefetched by
// cp.async one window ahead). Outputs 0..31 are final for the pass and go to A, outputs
// 32..63 go to cbuf[w&1] for window w+1: one __syncthreads per window orders everything
// (buffers alternate, so no window writes what the previous one may still read).
// NW = 8 warps (each 4 row tiles of one column tile; two CTAs fit an SM) or 16 (2 row
// tiles each; one CTA per SM, for grids too small to give every SM two CTAs).
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) rs_dmma_apply_kernel(double* __restrict__ A, long long m, long long lda,
                                                               int n, const double* __restrict__ qpass,
                                                               const unsigned long long* __restrict__ mpass,
                                                               int nwin) {
  extern __shared__ __align__(128) unsigned char dsm[];
  double* const qbuf = reinterpret_cast<double*>(dsm);  // 2 x kDQ (TMA, double buffered)
  double* const cbuf = qbuf + 2 * kDQ;                  // 2 x 32 columns x kDColStride (carried)
  double* const nbuf = cbuf + 2 * 32 * kDColStride;     // 2 x 32 columns x kDColStride (new)
  uint64_t* const qbar = reinterpret_cast<uint64_t*>(nbuf + 2 * 32 * kDColStride);
  constexpr int NT = NW * 32;
  constexpr int RT = 32 / NW;  // 8-row tiles per warp
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long r0 = (long long)blockIdx.x * kDRows;
  if (tid == 0) {
    mbar_init(&qbar[0], 1);
    mbar_init(&qbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // 32 columns starting at col0 into dst (one element per cp.async: any lda and alignment;
  // columns or rows outside the matrix are zero-filled)
  auto load_cols = [&](double* dst, int col0) {
#pragma unroll
    for (int it = 0; it < 32 * kDRows / NT; ++it) {
      const int idx = tid + it * NT;
      const int cl = idx >> 5, rr = idx & 31;
      const int col = col0 + cl;
      const long long row = r0 + rr;
      const bool ok = col >= 0 && col < n && row < m;
      cp_async_elem(dst + cl * kDColStride + rr, ok ? A + (long long)col * lda + row : A, ok);
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
  __syncthreads();
  // prologue: window 0's carried half (columns -31..0) and new half (1..32), Q_0
  load_cols(cbuf + 32 * kDColStride, -kDKB + 1);
  load_cols(nbuf, 1);
  issue_q(0);
  const int nt = warp & 7;         // this warp's 8 output columns of the window
  const int rt0 = (warp >> 3) * RT;  // and its first 8-row tile
  unsigned long long mask_next = __ldg(mpass);  // nonzero 8x8 tiles of Q_w
  for (int w = 0; w < nwin; ++w) {
    cp_async_wait_group<0>();  // this thread's copies for window w have landed
    __syncthreads();           // everyone's copies and window w-1's carried outputs; and
                               // every read of window w-1's buffers is done
    // prefetch the next window's new columns and Q_{w+1} into window w-1's buffers
    if (w + 1 < nwin) load_cols(nbuf + ((w + 1) & 1) * 32 * kDColStride, (w + 1) * kDNB + 1);
    issue_q(w + 1);
    mbar_wait(&qbar[w & 1], (uint32_t)(w >> 1) & 1u);
    const double* const qs = qbuf + (w & 1) * kDQ;
    const double* const xc = cbuf + ((w + 1) & 1) * 32 * kDColStride;  // window columns 0..31
    const double* const xn = nbuf + (w & 1) * 32 * kDColStride;        // window columns 32..63
    const unsigned long long mask = mask_next;
    if (w + 1 < nwin) mask_next = __ldg(mpass + w + 1);  // one window ahead: off the critical path
    // two accumulator sets (k-tiles 0..3 and 4..7 of the window) so every warp keeps eight
    // independent DMMA chains in flight; the k-steps of the two halves interleave
    double acc[2][RT][2];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) acc[hf][rt][0] = acc[hf][rt][1] = 0.0;
    auto kstep = [&](int hf, int ks) {  // one k-step (4 window columns) into acc[hf]
      const double b = qs[(ks * 8 + nt) * 32 + lane];
      const int kc = ks * 4 + (lane & 3);  // window column of this lane's A element
      const double* x =
          (hf == 0 ? xc + kc * kDColStride : xn + (kc - 32) * kDColStride) + rt0 * 8 + (lane >> 2);
      double a[RT];
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) a[rt] = x[rt * 8];
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) dmma884(acc[hf][rt], a[rt], b);
    };
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      const bool lo = (mask >> (kt * 8 + nt)) & 1ull;
      const bool hi = (mask >> ((kt + 4) * 8 + nt)) & 1ull;
      if (lo && hi) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          kstep(0, kt * 2 + h);
          kstep(1, (kt + 4) * 2 + h);
        }
      } else if (lo) {
        kstep(0, kt * 2);
        kstep(0, kt * 2 + 1);
      } else if (hi) {
        kstep(1, (kt + 4) * 2);
        kstep(1, (kt + 4) * 2 + 1);
      }
    }
#pragma unroll
    for (int rt = 0; rt < RT; ++rt) {
      acc[0][rt][0] += acc[1][rt][0];
      acc[0][rt][1] += acc[1][rt][1];
    }
    // outputs: window columns 0..31 are final for this pass (to A), 32..63 are carried
    double* const cout = cbuf + (w & 1) * 32 * kDColStride;
    const int ocol = nt * 8 + (lane & 3) * 2;  // window column of acc[.][0]
#pragma unroll
    for (int rt = 0; rt < RT; ++rt) {
      const int rr = (rt0 + rt) * 8 + (lane >> 2);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int wc = ocol + e;
        if (nt < 4) {
          const int col = w * kDNB - kDKB + 1 + wc;
          const long long row = r0 + rr;
          if (col >= 0 && col < n && row < m) A[(long long)col * lda + row] = acc[0][rt][e];
        } else {
          cout[(wc - 32) * kDColStride + rr] = acc[0][rt][e];
        }
      }
    }
  }
  cp_async_wait_group<0>();
  __syncthreads();
  // the last window's carried columns are final too
  {
    const double* const last = cbuf + ((nwin - 1) & 1) * 32 * kDColStride;
    const int col0 = nwin * kDNB - kDKB + 1;
    for (int idx = tid; idx < 32 * kDRows; idx += NT) {
      const int cl = idx / kDRows, rr = idx % kDRows;
      const int col = col0 + cl;
      const long long row = r0 + rr;
      if (col >= 0 && col < n && row < m) A[(long long)col * lda + row] = last[cl * kDColStride + rr];
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
  const size_t qsmem = sizeof(double2) * kDKB * kDPairs;
  static std::atomic<int> qconfigured{0};
  if (!qconfigured.load()) {
    if (cudaFuncSetAttribute(rs_dmma_q_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsmem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(rs_dmma_q_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsmem) !=
            cudaSuccess)
      return -1;
    qconfigured.store(1);
  }
  if (refl)
    rs_dmma_q_kernel<true><<<qg, kDW, qsmem, st>>>(q, masks, C, S, ldcs, (int)n, (int)k, rev);
  else
    rs_dmma_q_kernel<false><<<qg, kDW, qsmem, st>>>(q, masks, C, S, ldcs, (int)n, (int)k, rev);
  const size_t smem = (size_t)2 * kDQ * 8 + (size_t)4 * 32 * kDColStride * 8 + 2 * sizeof(uint64_t);
  static std::atomic<int> configured{0};
  if (!configured.load()) {
    if (cudaFuncSetAttribute(rs_dmma_apply_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(rs_dmma_apply_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
      return -1;
    configured.store(1);
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // reverse order: mirror the columns (base at the last column, negative stride)
  double* Ab = rev ? A + (long long)(n - 1) * lda : A;
  const long long ld = rev ? -lda : lda;
  const unsigned grid = (unsigned)((m + kDRows - 1) / kDRows);
  // measured (B200): 8-warp CTAs when the grid gives every SM two of them (65536 x 2048:
  // 22.4 vs 18.4 TF/s), 16-warp CTAs otherwise (4096^2: 15.0 vs 14.1 TF/s)
  const bool wide = grid < 2u * (unsigned)sms;
  for (int p = 0; p < passes; ++p) {
    if (wide)
      rs_dmma_apply_kernel<16><<<grid, 512, smem, st>>>(Ab, m, ld, (int)n, q + (size_t)p * nwin * kDQ,
                                                        masks + (size_t)p * nwin, nwin);
    else
      rs_dmma_apply_kernel<8><<<grid, 256, smem, st>>>(Ab, m, ld, (int)n, q + (size_t)p * nwin * kDQ,
                                                       masks + (size_t)p * nwin, nwin);
  }
  return cudaPeekAtLastError() == cudaSuccess ? passes + 1 : -1;
}

}  // namespace rsk
