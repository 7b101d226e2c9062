/*
 * oracle/rotseq_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference algorithm (package `rotseq`, arXiv 2412.01852
 * artifact, /root/reference/pkg/src/rotseq). It is the checker for the CUDA path and
 * the CPU baseline of bench.py; the product path never links, loads or calls it.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may use it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks these functions bit-for-bit against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py imports
 * /root/reference/pkg/src/rotseq and runs its strict build).
 *
 * Compiled twice from this one source, mirroring the reference's dual build
 * (_jit.py:14-15, 26-44):
 *   ORACLE_FAST=0, -ffp-contract=off  -> *_strict  (plain IEEE; bit-identical to the
 *                                        reference strict build)
 *   ORACLE_FAST=1, -ffp-contract=fast -> *_fast    (FMA contraction allowed)
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if ORACLE_FAST
#define FN(name) name##_fast
#else
#define FN(name) name##_strict
#endif

#define HOT __attribute__((target_clones("avx512f", "avx2", "default")))

/* ------------------------------------------------------------------------------------
 * 2x2 kernels on strided line pairs.
 *   rotation  (core.py:130-137): t = c*x + s*y; y' = c*y - s*x; x' = t
 *   reflector (core.py:140-149): d = c-s; e = c+s; w = s*(x+y); x' = w + d*x; y' = w - e*y
 * ------------------------------------------------------------------------------------ */
HOT static void rot_lines(double* restrict x, double* restrict y, int64_t cnt, int64_t es, double c, double s) {
  if (es == 1) {
    for (int64_t i = 0; i < cnt; ++i) {
      const double xv = x[i], yv = y[i];
      const double t = c * xv + s * yv;
      y[i] = c * yv - s * xv;
      x[i] = t;
    }
  } else {
    for (int64_t i = 0; i < cnt; ++i) {
      const double xv = x[i * es], yv = y[i * es];
      const double t = c * xv + s * yv;
      y[i * es] = c * yv - s * xv;
      x[i * es] = t;
    }
  }
}

HOT static void refl_lines(double* restrict x, double* restrict y, int64_t cnt, int64_t es, double c, double s) {
  const double d = c - s;
  const double e = c + s;
  if (es == 1) {
    for (int64_t i = 0; i < cnt; ++i) {
      const double xv = x[i], yv = y[i];
      const double w = s * (xv + yv);
      x[i] = w + d * xv;
      y[i] = w - e * yv;
    }
  } else {
    for (int64_t i = 0; i < cnt; ++i) {
      const double xv = x[i * es], yv = y[i * es];
      const double w = s * (xv + yv);
      x[i * es] = w + d * xv;
      y[i * es] = w - e * yv;
    }
  }
}

/* ------------------------------------------------------------------------------------
 * Semantic definition: _naive_py (core.py:195-205), for p < k: for j < len-1.
 * Extensions (not in the reference):
 *   side = 1 (left): the pair is rows (j, j+1) instead of columns; C/S are (m-1) x k.
 *   order = 1 (reverse): inside each sweep p, j runs len-2 down to 0.
 * The 2x2 arithmetic is unchanged, so both are pinned to the reference by the exact
 * identities left(A) = right(A^T)^T and reverse(A; C, S) = mirror(right(mirror(A); C', -S'))
 * (tests/golden/make_golden.py generates those goldens with the reference itself).
 * ------------------------------------------------------------------------------------ */
void FN(oracle_apply_naive_f64)(double* A, int64_t m, int64_t n, int64_t lda, const double* C, const double* S,
                                int64_t ldcs, int64_t k, int side, int order, int kind, int64_t owner0,
                                int64_t owner1) {
  const int left = side == 1;
  const int64_t len = left ? m : n;
  const int64_t pair_stride = left ? 1 : lda; /* line j -> line j+1 */
  const int64_t es = left ? lda : 1;         /* owner i -> owner i+1 */
  if (owner1 <= owner0) return;
  double* base = A + owner0 * es;
  const int64_t cnt = owner1 - owner0;
  for (int64_t p = 0; p < k; ++p) {
    for (int64_t jj = 0; jj < len - 1; ++jj) {
      const int64_t j = order ? len - 2 - jj : jj;
      const double c = C[j + p * ldcs];
      const double s = S[j + p * ldcs];
      double* x = base + j * pair_stride;
      double* y = x + pair_stride;
      if (kind == 1)
        refl_lines(x, y, cnt, es, c, s);
      else
        rot_lines(x, y, cnt, es, c, s);
    }
  }
}

/* ------------------------------------------------------------------------------------
 * Kernel tier (the reference's fastest CPU path, algo "kernel"): apply_blocked with
 * use_kernel=True (blocking.py:420-476): row blocks of m_b rows packed into m_r-row
 * panels (blocking.py:249-299), sequence chunks of width min(k_b, n-1)
 * (blocking.py:408-417), and per chunk _kernel_chunk_py (blocking.py:342-397): startup
 * triangle, windows of n_b waves with wave-major coefficient tiles, shutdown triangle;
 * then unpack (blocking.py:263-272, 302-312). Threads over row ranges as
 * partition_rows / _run_row_ranges (blocking.py:178-202, 518-526). Right side, forward
 * order (the reference's only semantics). Bit-identical to the naive loop in strict mode.
 * ------------------------------------------------------------------------------------ */
HOT static void rot_panel(double* restrict P, int64_t m_r, int64_t j, double c, double s) {
  double* restrict x = P + j * m_r;
  double* restrict y = P + (j + 1) * m_r;
  for (int64_t i = 0; i < m_r; ++i) {
    const double xv = x[i], yv = y[i];
    const double t = c * xv + s * yv;
    y[i] = c * yv - s * xv;
    x[i] = t;
  }
}

HOT static void refl_panel(double* restrict P, int64_t m_r, int64_t j, double c, double s) {
  const double d = c - s;
  const double e = c + s;
  double* restrict x = P + j * m_r;
  double* restrict y = P + (j + 1) * m_r;
  for (int64_t i = 0; i < m_r; ++i) {
    const double xv = x[i], yv = y[i];
    const double w = s * (xv + yv);
    x[i] = w + d * xv;
    y[i] = w - e * yv;
  }
}

static void kernel_chunk(double* P3, int64_t n_panels, int64_t n, int64_t m_r, const double* C, const double* S,
                         int64_t ldcs, int64_t p0, int64_t kw, int64_t n_b, int64_t k_r, int refl, double* ct,
                         double* st) {
  const int64_t pstride = n * m_r;
  /* startup triangle (blocking.py:348-356) */
  for (int64_t q = 0; q < n_panels; ++q) {
    double* P = P3 + q * pstride;
    for (int64_t pp = 0; pp < kw - 1; ++pp) {
      const int64_t p = p0 + pp;
      for (int64_t row = 0; row < kw - 1 - pp; ++row) {
        if (refl)
          refl_panel(P, m_r, row, C[row + p * ldcs], S[row + p * ldcs]);
        else
          rot_panel(P, m_r, row, C[row + p * ldcs], S[row + p * ldcs]);
      }
    }
  }
  /* pipeline windows (blocking.py:357-388) */
  const int64_t nL = (kw + k_r - 1) / k_r;
  for (int64_t t0 = kw - 1; t0 < n - 1; t0 += n_b) {
    int64_t nw = n - 1 - t0;
    if (nw > n_b) nw = n_b;
    for (int64_t l = 0; l < nL; ++l) {
      int64_t kr_l = kw - l * k_r;
      if (kr_l > k_r) kr_l = k_r;
      const int64_t pl = p0 + l * k_r;
      for (int64_t w = 0; w < nw; ++w)
        for (int64_t lam = 0; lam < kr_l; ++lam) {
          const int64_t row = t0 + w - l * k_r - lam;
          ct[l * n_b * k_r + w * kr_l + lam] = C[row + (pl + lam) * ldcs];
          st[l * n_b * k_r + w * kr_l + lam] = S[row + (pl + lam) * ldcs];
        }
    }
    for (int64_t q = 0; q < n_panels; ++q) {
      double* P = P3 + q * pstride;
      for (int64_t l = 0; l < nL; ++l) {
        int64_t kr_l = kw - l * k_r;
        if (kr_l > k_r) kr_l = k_r;
        const int64_t col0 = t0 - l * k_r - (kr_l - 1);
        for (int64_t w = 0; w < nw; ++w) {
          const int64_t base = w * kr_l;
          for (int64_t lam = 0; lam < kr_l; ++lam) {
            const int64_t j = col0 + w + kr_l - 1 - lam;
            const double c = ct[l * n_b * k_r + base + lam];
            const double s = st[l * n_b * k_r + base + lam];
            if (refl)
              refl_panel(P, m_r, j, c, s);
            else
              rot_panel(P, m_r, j, c, s);
          }
        }
      }
    }
  }
  /* shutdown triangle (blocking.py:389-397) */
  for (int64_t q = 0; q < n_panels; ++q) {
    double* P = P3 + q * pstride;
    for (int64_t pp = 1; pp < kw; ++pp) {
      const int64_t p = p0 + pp;
      for (int64_t row = n - 1 - pp; row < n - 1; ++row) {
        if (refl)
          refl_panel(P, m_r, row, C[row + p * ldcs], S[row + p * ldcs]);
        else
          rot_panel(P, m_r, row, C[row + p * ldcs], S[row + p * ldcs]);
      }
    }
  }
}

typedef struct {
  double* A;
  int64_t n, lda;
  const double* C;
  const double* S;
  int64_t ldcs, k;
  int refl;
  int64_t n_b, k_b, m_b, m_r, k_r;
  int64_t r0, r1;
  int status;
} blocked_job;

static void* blocked_worker(void* arg) {
  blocked_job* jb = (blocked_job*)arg;
  const int64_t n = jb->n, m_r = jb->m_r;
  const int64_t cap = jb->k_b < n - 1 ? jb->k_b : n - 1; /* _chunk_widths, blocking.py:408-417 */
  const int64_t max_panels = (jb->m_b + m_r - 1) / m_r;
  double* P3 = (double*)aligned_alloc(64, ((size_t)(max_panels * n * m_r * sizeof(double)) + 63) / 64 * 64);
  const int64_t nL = (cap + jb->k_r - 1) / jb->k_r;
  double* ct = (double*)malloc(sizeof(double) * (size_t)(nL * jb->n_b * jb->k_r + 1));
  double* st = (double*)malloc(sizeof(double) * (size_t)(nL * jb->n_b * jb->k_r + 1));
  if (!P3 || !ct || !st) {
    jb->status = 1;
    free(P3);
    free(ct);
    free(st);
    return NULL;
  }
  for (int64_t rb = jb->r0; rb < jb->r1; rb += jb->m_b) {
    int64_t rc = jb->r1 - rb;
    if (rc > jb->m_b) rc = jb->m_b;
    const int64_t n_panels = (rc + m_r - 1) / m_r;
    /* pack (blocking.py:249-260): zero-padded m_r-row panels */
    for (int64_t q = 0; q < n_panels; ++q) {
      int64_t h = rc - q * m_r;
      if (h > m_r) h = m_r;
      for (int64_t j = 0; j < n; ++j) {
        double* dst = P3 + (q * n + j) * m_r;
        const double* src = jb->A + rb + q * m_r + j * jb->lda;
        memcpy(dst, src, sizeof(double) * (size_t)h);
        for (int64_t i = h; i < m_r; ++i) dst[i] = 0.0;
      }
    }
    for (int64_t p0 = 0; p0 < jb->k; p0 += cap) {
      int64_t kw = jb->k - p0;
      if (kw > cap) kw = cap;
      kernel_chunk(P3, n_panels, n, m_r, jb->C, jb->S, jb->ldcs, p0, kw, jb->n_b, jb->k_r, jb->refl, ct, st);
    }
    /* unpack (blocking.py:263-272) */
    for (int64_t q = 0; q < n_panels; ++q) {
      int64_t h = rc - q * m_r;
      if (h > m_r) h = m_r;
      for (int64_t j = 0; j < n; ++j)
        memcpy(jb->A + rb + q * m_r + j * jb->lda, P3 + (q * n + j) * m_r, sizeof(double) * (size_t)h);
    }
  }
  free(P3);
  free(ct);
  free(st);
  jb->status = 0;
  return NULL;
}

/* partition_rows (blocking.py:178-202): balanced m_r-multiple ranges; the leftover
 * rows below one unit go to the last populated range. */
void FN(oracle_partition_rows)(int64_t m, int64_t threads, int64_t m_r, int64_t* out_ranges) {
  const int64_t units = m / m_r, rem = m % m_r;
  const int64_t base = units / threads, extra = units % threads;
  int64_t last = 0;
  for (int64_t i = 0; i < threads; ++i) {
    const int64_t ln = (base + (i < extra ? 1 : 0)) * m_r;
    out_ranges[2 * i + 1] = ln;
    if (ln > 0) last = i;
  }
  out_ranges[2 * last + 1] += rem;
  int64_t start = 0;
  for (int64_t i = 0; i < threads; ++i) {
    const int64_t ln = out_ranges[2 * i + 1];
    out_ranges[2 * i] = start;
    out_ranges[2 * i + 1] = start + ln;
    start += ln;
  }
}

int FN(oracle_apply_blocked_f64)(double* A, int64_t m, int64_t n, int64_t lda, const double* C, const double* S,
                                 int64_t ldcs, int64_t k, int kind, int64_t n_b, int64_t k_b, int64_t m_b,
                                 int64_t m_r, int64_t k_r, int threads) {
  if (m <= 0) return 0;
  if (n < 2 || k < 1 || n_b < 1 || k_b < 1 || m_b < 1 || m_r < 1 || k_r < 1 || threads < 1) return 2;
  int64_t* ranges = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)threads);
  blocked_job* jobs = (blocked_job*)calloc((size_t)threads, sizeof(blocked_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  if (!ranges || !jobs || !tids) return 1;
  if (threads == 1) {
    ranges[0] = 0;
    ranges[1] = m;
  } else {
    FN(oracle_partition_rows)(m, threads, m_r, ranges);
  }
  int rc = 0;
  char* created = (char*)calloc((size_t)threads, 1);
  if (!created) return 1;
  for (int i = 0; i < threads; ++i) {
    blocked_job* jb = &jobs[i];
    jb->A = A;
    jb->n = n;
    jb->lda = lda;
    jb->C = C;
    jb->S = S;
    jb->ldcs = ldcs;
    jb->k = k;
    jb->refl = kind == 1;
    jb->n_b = n_b;
    jb->k_b = k_b;
    jb->m_b = m_b;
    jb->m_r = m_r;
    jb->k_r = k_r;
    jb->r0 = ranges[2 * i];
    jb->r1 = ranges[2 * i + 1];
    jb->status = 0;
    if (jb->r1 <= jb->r0) continue;
    if (threads == 1) {
      blocked_worker(jb);
    } else if (pthread_create(&tids[i], NULL, blocked_worker, jb) != 0) {
      blocked_worker(jb);
    } else {
      created[i] = 1;
    }
  }
  for (int i = 0; i < threads; ++i)
    if (created[i]) pthread_join(tids[i], NULL);
  for (int i = 0; i < threads; ++i)
    if (jobs[i].status > 0) rc = 1;
  free(created);
  free(ranges);
  free(jobs);
  free(tids);
  return rc;
}
