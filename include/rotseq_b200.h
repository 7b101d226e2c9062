/*
 * rotseq_b200 — C-ABI of the B200-native rotation-sequence apply.
 *
 * Drop-in boundary for the reference package `rotseq` (arXiv 2412.01852 artifact):
 *
 *   reference entry point                         replaced by
 *   --------------------------------------------  ------------------------------------
 *   rotseq.core.apply_naive(A, seq, kind, fast)    rs_apply_f64(..., side=0, order=0, ...)
 *     /root/reference/pkg/src/rotseq/core.py:365-374
 *   rotseq.blocking.apply_blocked(A, seq, plan,    rs_apply_f64(...)   (plan/shape/threads are
 *     shape, kind, threads, fast, use_kernel)        CPU cache knobs; the GPU tiling is internal)
 *     /root/reference/pkg/src/rotseq/blocking.py:420-476
 *   rotseq.verification.run_variant("kernel",...)  run_variant("cuda", ...) in the Python mirror
 *     /root/reference/pkg/src/rotseq/verification.py:50-85
 *   rotseq.blocking._kernel_chunk (the hot loop)   rs_pipeline kernel (internal)
 *     /root/reference/pkg/src/rotseq/blocking.py:342-397
 *
 * Semantics (reference core.py:1-16, 130-149, 195-205):
 *   A is an m x n column-major matrix (element (i,j) at A[i + j*lda]).
 *   C and S are (len-1) x k column-major with leading dimension ldcs, where len = n for
 *   side = RS_SIDE_RIGHT and len = m for side = RS_SIDE_LEFT.
 *   For p = 0..k-1 (sweeps, ascending) and j = 0..len-2 (ascending; descending when
 *   order = RS_ORDER_REVERSE), the 2x2 transform with (c, s) = (C[j,p], S[j,p]) is
 *   applied to the pair x = column j, y = column j+1 (right side) or x = row j,
 *   y = row j+1 (left side):
 *     rotation : x' = c*x + s*y ;  y' = c*y - s*x            (core.py:130-137)
 *     reflector: w = s*(x+y) ; x' = w + (c-s)*x ; y' = w - (c+s)*y   (core.py:140-149)
 *   strict != 0: plain IEEE mul/add in exactly that expression shape (no FMA
 *   contraction) -> bit-identical to the reference's strict numba build (_jit.py:14).
 *   strict == 0: FMA contraction allowed (the reference's "fast" build, _jit.py:15).
 *
 * All pointers are DEVICE pointers. Calls are asynchronous on `stream` (a cudaStream_t,
 * NULL = legacy default stream) and thread-safe for distinct buffers / workspaces.
 * The library never frees caller buffers. A, C, S are owned by the caller.
 *
 * Errors: functions return rs_status; rs_last_error() returns a thread-local message
 * for the last failing call on the calling thread. The Python mirror maps RS_EINVAL to
 * ValueError (the reference raises ValueError for every argument error, core.py:41-51,
 * 110-117) and everything else to RuntimeError.
 */
#ifndef ROTSEQ_B200_H
#define ROTSEQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RS_OK = 0,
  RS_EINVAL = 1,       /* bad argument (shape, stride, enum, null pointer)        */
  RS_ECUDA = 2,        /* CUDA runtime error (launch failure, no device, ...)     */
  RS_ENOMEM = 3,       /* workspace too small / allocation failed                 */
  RS_EUNSUPPORTED = 4  /* configuration this build does not provide               */
} rs_status;

enum { RS_SIDE_RIGHT = 0, RS_SIDE_LEFT = 1 };
enum { RS_ORDER_FORWARD = 0, RS_ORDER_REVERSE = 1 };
enum { RS_KIND_ROTATION = 0, RS_KIND_REFLECTOR = 1 };
enum { RS_DTYPE_F64 = 0, RS_DTYPE_F32 = 1 };
enum { RS_ALGO_PIPELINE = 0, RS_ALGO_NAIVE = 1 };

/* Library / ABI version (major*10000 + minor*100 + patch). */
int rs_version(void);

/* Thread-local message describing the last error on this thread ("" if none). */
const char* rs_last_error(void);

/* Bytes of device workspace rs_apply_* needs for this problem (packed coefficients +
 * inter-CTA progress flags). Passing workspace == NULL to rs_apply_* makes the library
 * allocate (and stream-order free) it itself. Returns 0 on invalid arguments. */
size_t rs_workspace_bytes(int64_t m, int64_t n, int64_t k, int side, int kind, int dtype);

/* Apply the rotation sequence (C, S) to A in place (see header comment).
 * Replaces rotseq.core.apply_naive / rotseq.blocking.apply_blocked
 * (core.py:365-374, blocking.py:420-476). */
rs_status rs_apply_f64(double* A, int64_t m, int64_t n, int64_t lda,
                       const double* C, const double* S, int64_t ldcs, int64_t k,
                       int side, int order, int kind, int strict,
                       void* workspace, size_t workspace_bytes, void* stream);

/* fp32 instantiation (BASELINE config 4). Same contract; tolerance-checked against the
 * reference run in fp64 on the same fp32-rounded inputs. */
rs_status rs_apply_f32(float* A, int64_t m, int64_t n, int64_t lda,
                       const float* C, const float* S, int64_t ldcs, int64_t k,
                       int side, int order, int kind, int strict,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Same as rs_apply_* with an explicit algorithm: RS_ALGO_PIPELINE (the product
 * register-window band pipeline) or RS_ALGO_NAIVE (one thread per row/column, plain
 * sweep loop in global memory: the GPU restatement of _naive_py, core.py:195-205, kept
 * as an independent second implementation for cross-checks). */
rs_status rs_apply_algo_f64(int algo, double* A, int64_t m, int64_t n, int64_t lda,
                            const double* C, const double* S, int64_t ldcs, int64_t k,
                            int side, int order, int kind, int strict,
                            void* workspace, size_t workspace_bytes, void* stream);
rs_status rs_apply_algo_f32(int algo, float* A, int64_t m, int64_t n, int64_t lda,
                            const float* C, const float* S, int64_t ldcs, int64_t k,
                            int side, int order, int kind, int strict,
                            void* workspace, size_t workspace_bytes, void* stream);

/* Prepacked / resident mode (the reference's apply_blocked_packed, blocking.py:479-515,
 * and the paper's rs_kernel_v2): rs_pack_* repacks C/S into the caller's workspace
 * (rs_workspace_bytes() bytes, 256-byte aligned) as the band-major, wave-major coefficient
 * stream the kernel consumes; rs_apply_packed_* then applies it to A any number of times
 * without touching C/S again. (m, n, k, side, order, kind) must match between the two.
 * rs_apply_* is exactly rs_pack_* followed by rs_apply_packed_*. */
rs_status rs_pack_f64(const double* C, const double* S, int64_t ldcs, int64_t m, int64_t n, int64_t k,
                      int side, int order, int kind, void* workspace, size_t workspace_bytes, void* stream);
rs_status rs_pack_f32(const float* C, const float* S, int64_t ldcs, int64_t m, int64_t n, int64_t k,
                      int side, int order, int kind, void* workspace, size_t workspace_bytes, void* stream);
/* Fast-mode-only pack: as rs_pack_*, but the standard (unscaled) records are written only
 * when the scaled form is out of range for these coefficients — the per-call fast path's
 * pack. The workspace may then only be applied with strict = 0 (the Python mirror,
 * PackedSequence(fast_only=True), enforces it). */
rs_status rs_pack_fast_f64(const double* C, const double* S, int64_t ldcs, int64_t m, int64_t n, int64_t k,
                           int side, int order, int kind, void* workspace, size_t workspace_bytes, void* stream);
rs_status rs_pack_fast_f32(const float* C, const float* S, int64_t ldcs, int64_t m, int64_t n, int64_t k,
                           int side, int order, int kind, void* workspace, size_t workspace_bytes, void* stream);
rs_status rs_apply_packed_f64(double* A, int64_t m, int64_t n, int64_t lda, int64_t k, int side, int order,
                              int kind, int strict, void* workspace, size_t workspace_bytes, void* stream);
rs_status rs_apply_packed_f32(float* A, int64_t m, int64_t n, int64_t lda, int64_t k, int side, int order,
                              int kind, int strict, void* workspace, size_t workspace_bytes, void* stream);

/* Arithmetic form a fast-mode rs_apply_packed_* will use with this packed workspace
 * (after rs_pack_* / rs_pack_fast_* on `stream`; synchronous): *scaled_units of the
 * *total_units (tile, sweep-range) units run the scaled "fast Givens" form (2 FMAs per
 * rotation element), the rest the standard fast form (2 MUL + 2 FMA) because their
 * coefficients leave the scaled form's safe range (e.g. c == 0). Strict applies always
 * use the reference's expression shape. Reference: the strict/fast contract, _jit.py:14-44. */
rs_status rs_packed_form(const void* workspace, size_t workspace_bytes, int64_t m, int64_t n, int64_t k,
                         int side, int kind, int dtype, int64_t* scaled_units, int64_t* total_units,
                         void* stream);

/* Host-buffer entry point: A (m x n, column-major, lda), C and S ((len-1) x k, ldcs) in
 * HOST memory (pinned for full bandwidth; pageable works, slower). Synchronous: returns
 * once A holds the result. This is the call a host-side binding of the reference makes
 * in place of rotseq.core.apply_naive / rotseq.blocking.apply_blocked
 * (core.py:365-374, blocking.py:420-476) when its data lives in host memory: C/S are
 * copied and packed, then A streams in and out in wave-column chunks that overlap with
 * the pipeline kernel (copy-in, compute and copy-out run concurrently). Device buffers
 * come from the stream-ordered allocator; `stream` orders the compute. */
rs_status rs_apply_host_f64(double* A, int64_t m, int64_t n, int64_t lda,
                            const double* C, const double* S, int64_t ldcs, int64_t k,
                            int side, int order, int kind, int strict, void* stream);
rs_status rs_apply_host_f32(float* A, int64_t m, int64_t n, int64_t lda,
                            const float* C, const float* S, int64_t ldcs, int64_t k,
                            int side, int order, int kind, int strict, void* stream);

/* Micro-kernel API (the reference's kernel_wave_apply, kernels.py:335-371): apply n_waves
 * waves of k_r transforms to a panel of m_r rows and n_cols columns, column j at
 * panel + j*ld with its m_r rows contiguous (the reference's C-contiguous (n_cols, m_r)
 * panel is ld = m_r). Wave w, lane l rotates columns (col0 + w + k_r - 1 - l, +1) with
 * ct[w*k_r + l], st[w*k_r + l] (wave-major tiles, kernels.py:12-13). Requires
 * n_cols - col0 >= n_waves + k_r. Strict arithmetic is bit-identical to the reference's
 * strict build; device pointers, asynchronous on `stream`. kernel_edge_apply
 * (kernels.py:374-410) is a sequence of k_r = 1 calls. */
rs_status rs_wave_apply_f64(double* panel, int64_t m_r, int64_t n_cols, int64_t ld, const double* ct,
                            const double* st, int64_t n_waves, int64_t k_r, int64_t col0, int kind, int strict,
                            void* stream);
rs_status rs_wave_apply_f32(float* panel, int64_t m_r, int64_t n_cols, int64_t ld, const float* ct,
                            const float* st, int64_t n_waves, int64_t k_r, int64_t col0, int kind, int strict,
                            void* stream);

/* The accumulate-and-apply variant on the FP64 tensor cores (the paper's rs_gemm,
 * PAPER.md:860; explicit-Q idea of accumulate_q, oracle.py:102-109): the k sweeps in passes
 * of 32, each pass's rotations grouped into 64 x 64 window products Q_w (32 waves each)
 * that are applied as A[:, window] <- A[:, window] * Q_w with DMMA (mma.sync m8n8k4 f64).
 * Right side, either order and kind, fp64, fast-mode accuracy (within the BASELINE
 * tolerance, not bit-identical). Device pointers; asynchronous on `stream`; `workspace`
 * (rs_dmma_workspace_bytes(), 256-byte aligned) may be NULL (stream-ordered allocation). */
size_t rs_dmma_workspace_bytes(int64_t m, int64_t n, int64_t k);
rs_status rs_apply_dmma_f64(double* A, int64_t m, int64_t n, int64_t lda, const double* C, const double* S,
                            int64_t ldcs, int64_t k, int order, int kind, void* workspace, size_t workspace_bytes,
                            void* stream);

/* Launch geometry the pipeline would use for this problem on the current device
 * (for benchmarks / roofline accounting). Any out-pointer may be NULL. */
rs_status rs_plan_info(int64_t m, int64_t n, int64_t k, int side, int kind, int dtype,
                       int* grid_ctas, int* warps_per_cta, int64_t* units, int* band_width,
                       int* rows_per_tile, size_t* smem_bytes);

/* The compile-time tile shape of the pipeline kernel for (dtype, side): sweeps per unit
 * window (the reference's k_r), rows per thread (tile rows = 32 * rows_per_thread, the
 * reference's m_r), ring depth in chunks, and the warps-per-CTA bounds of the two register
 * budgets the kernel is built for (a build for at most `small_cta_warps` warps, 0 if the
 * family has none, and one for up to `max_warps`). Needs no GPU; the host-side tile model
 * (paper_2412_01852_b200/model.py, the counterpart of the reference's choose_block_sizes,
 * blocking.py:115-147) must choose exactly these values. Any out-pointer may be NULL. */
rs_status rs_tile_shape(int dtype, int side, int* window_sweeps, int* rows_per_thread, int* ring_chunks,
                        int* small_cta_warps, int* max_warps);

/* Measured FMA-pipe peak of the current device (TFLOP/s, 2 flops per FMA) for dtype
 * RS_DTYPE_F64 (DFMA) or RS_DTYPE_F32 (FFMA): the roofline denominator for this
 * FP-bound path. Synchronous (~10 ms). Not on the apply path. */
rs_status rs_fma_peak_tflops(int dtype, double* tflops, void* stream);

/* Number of pipeline / pack / naive kernel launches issued by this library since
 * process start (all threads). Used by bench.py to report gpu_launches. */
int64_t rs_launch_count(void);

/* Debug only (library built with -DRS_TRACE, else RS_EUNSUPPORTED): install (non-NULL)
 * or remove (NULL) a device-visible buffer of grid*16*32*10 uint64 words that the
 * pipeline kernel fills with one record per unit (start/end time, wait/compute cycle
 * breakdown) for timeline analysis. */
rs_status rs_debug_set_trace(void* device_ptr);

#ifdef __cplusplus
}
#endif

#endif /* ROTSEQ_B200_H */
