/*
 * fk_oracle.c -- CPU restatement of the flashmeans hot path (TEST INFRASTRUCTURE).
 *
 * THIS FILE IS THE PARITY ORACLE, NOT PRODUCT CODE.  Only tests/, the
 * __graft_entry__.smoke() checker and bench.py's cpu_baseline / --impl
 * reference leg may load it.  The product path (paper_2603_09229_b200) never
 * links, imports or calls anything under oracle/.
 *
 * It restates, in plain C, the arithmetic of the reference package
 * flashmeans 0.1.0 (/root/reference/pkg/src/flashmeans) bit for bit:
 *
 *   orc_row_norms_*      <- _kernels.row_norms_acc        _kernels.py:21-29
 *                           + core.row_norms astype        core.py:307-318
 *   orc_assign_*         <- _kernels.dist_block            _kernels.py:32-45
 *                           + _kernels.rowmin_merge        _kernels.py:64-82
 *                           driven by flash_assign         flash_assign.py:135-222
 *   orc_counting_sort    <- _kernels.counting_sort         _kernels.py:118-132
 *   orc_sort_inverse_*   <- sort_inverse_update            sort_inverse.py:106-149
 *                           + segment_stats / merge_segments _kernels.py:135-171
 *   orc_scatter_*        <- _kernels.scatter_rows          _kernels.py:107-115
 *   orc_normalize_*      <- baseline.normalize             baseline.py:127-150
 *
 * Precision rules (pinned against the live reference by
 * tests/test_oracle_reference.py and tests/golden/):
 *   xn_i   = fl_T( sum_{j asc} fl64( fl_T(x_ij * x_ij) ) )
 *   acc_ik = sum_{j asc} fl64( fl_T(x_ij * c_kj) )
 *   D_ik   = fl_T( max(0, fl64(fl_T(xn_i + cn_k)) - 2*acc_ik) )
 *   a_i    = lowest k with D_ik == min_k D_ik   (strict < in ascending k)
 * Build with -ffp-contract=off: no FMA contraction anywhere.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

ORC_API int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------- norms */
ORC_API void orc_row_norms_f32(const float* m, int64_t n, int64_t d, float* out) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    const float* r = m + i * d;
    for (int64_t j = 0; j < d; ++j) {
      float p = r[j] * r[j];          /* f32 product (numba: f32*f32 -> f32) */
      acc += (double)p;               /* f64 accumulator */
    }
    out[i] = (float)acc;              /* astype(float32) */
  }
}

ORC_API void orc_row_norms_f64(const double* m, int64_t n, int64_t d, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    const double* r = m + i * d;
    for (int64_t j = 0; j < d; ++j) acc += r[j] * r[j];
    out[i] = acc;
  }
}

/* ---------------------------------------------------------------- assign */
/* One batch element.  a[i], m[i] for i in [0,N).  Mirrors flash_assign in
 * dot_mode="exact": tile shape does not matter (flash_assign.py:12-14), so a
 * single ascending sweep over k with strict < is the same decision rule.  */
ORC_API void orc_assign_f32(const float* X, const float* C, int64_t N, int64_t K, int64_t d,
                            int32_t* a, float* m, int threads) {
  float* xn = (float*)malloc(sizeof(float) * (size_t)(N > 0 ? N : 1));
  float* cn = (float*)malloc(sizeof(float) * (size_t)(K > 0 ? K : 1));
  orc_row_norms_f32(X, N, d, xn);
  orc_row_norms_f32(C, K, d, cn);
#ifdef _OPENMP
  if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
#endif
  for (int64_t i = 0; i < N; ++i) {
    const float* x = X + i * d;
    float best = INFINITY;
    int32_t bi = -1;
    for (int64_t k = 0; k < K; ++k) {
      const float* c = C + k * d;
      double acc = 0.0;
      for (int64_t j = 0; j < d; ++j) {
        float p = x[j] * c[j];
        acc += (double)p;
      }
      float s = xn[i] + cn[k];                   /* f32 + f32 */
      double v = (double)s - 2.0 * acc;          /* promoted to f64 */
      if (v < 0.0) v = 0.0;
      float vf = (float)v;                       /* stored in the f32 block */
      if (vf < best) { best = vf; bi = (int32_t)k; }
    }
    a[i] = bi;
    m[i] = best;
  }
  free(xn);
  free(cn);
}

ORC_API void orc_assign_f64(const double* X, const double* C, int64_t N, int64_t K, int64_t d,
                            int32_t* a, double* m, int threads) {
  double* xn = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
  double* cn = (double*)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
  orc_row_norms_f64(X, N, d, xn);
  orc_row_norms_f64(C, K, d, cn);
#ifdef _OPENMP
  if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
#endif
  for (int64_t i = 0; i < N; ++i) {
    const double* x = X + i * d;
    double best = INFINITY;
    int32_t bi = -1;
    for (int64_t k = 0; k < K; ++k) {
      const double* c = C + k * d;
      double acc = 0.0;
      for (int64_t j = 0; j < d; ++j) acc += x[j] * c[j];
      double v = (xn[i] + cn[k]) - 2.0 * acc;
      if (v < 0.0) v = 0.0;
      if (v < best) { best = v; bi = (int32_t)k; }
    }
    a[i] = bi;
    m[i] = best;
  }
  free(xn);
  free(cn);
}

/* ---------------------------------------------------------- sort-inverse */
/* Stable counting sort of ids (one batch element): _kernels.py:118-132.  */
ORC_API void orc_counting_sort(const int32_t* ids, int64_t N, int64_t K, int64_t* order,
                               int32_t* a_sorted) {
  int64_t* off = (int64_t*)calloc((size_t)K + 1, sizeof(int64_t));
  for (int64_t i = 0; i < N; ++i) off[ids[i] + 1] += 1;
  for (int64_t j = 0; j < K; ++j) off[j + 1] += off[j];
  for (int64_t i = 0; i < N; ++i) {
    int32_t key = ids[i];
    int64_t pos = off[key]++;
    order[pos] = i;
    a_sorted[pos] = key;
  }
  free(off);
}

/* sort_inverse_update for one batch element (sort_inverse.py:106-149).
 * X is f32 (is_f64=0) or f64 (is_f64=1).  sums (K,d) f64 and counts (K) i64
 * are ACCUMULATED into (the caller zeroes them), exactly like merge_segments.
 * Returns the number of segments merged (synchronized_merges increment). */
static int64_t sort_inverse_impl(const void* X, int is_f64, const int32_t* ids, int64_t N,
                                 int64_t K, int64_t d, int64_t chunk, double* sums,
                                 int64_t* counts) {
  if (N == 0) return 0;
  if (chunk < 1) chunk = 1;
  if (chunk > N) chunk = N;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  int32_t* a_sorted = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
  orc_counting_sort(ids, N, K, order, a_sorted);
  double* seg = (double*)malloc(sizeof(double) * (size_t)d);
  int64_t merges = 0;
  for (int64_t lo = 0; lo < N; lo += chunk) {
    int64_t hi = lo + chunk < N ? lo + chunk : N;
    int64_t t = lo;
    while (t < hi) {                         /* one segment = maximal run in chunk */
      int32_t key = a_sorted[t];
      int64_t cnt = 0;
      for (int64_t j = 0; j < d; ++j) seg[j] = 0.0;
      while (t < hi && a_sorted[t] == key) {
        int64_t row = order[t];
        if (is_f64) {
          const double* r = (const double*)X + row * d;
          for (int64_t j = 0; j < d; ++j) seg[j] += r[j];
        } else {
          const float* r = (const float*)X + row * d;
          for (int64_t j = 0; j < d; ++j) seg[j] += (double)r[j];
        }
        cnt += 1;
        t += 1;
      }
      /* merge_segments: sums[k] += seg (ascending segment order) */
      double* dst = sums + (int64_t)key * d;
      for (int64_t j = 0; j < d; ++j) dst[j] += seg[j];
      counts[key] += cnt;
      merges += 1;
    }
  }
  free(seg);
  free(order);
  free(a_sorted);
  return merges;
}

ORC_API int64_t orc_sort_inverse_f32(const float* X, const int32_t* ids, int64_t N, int64_t K,
                                     int64_t d, int64_t chunk, double* sums, int64_t* counts) {
  return sort_inverse_impl(X, 0, ids, N, K, d, chunk, sums, counts);
}

ORC_API int64_t orc_sort_inverse_f64(const double* X, const int32_t* ids, int64_t N, int64_t K,
                                     int64_t d, int64_t chunk, double* sums, int64_t* counts) {
  return sort_inverse_impl(X, 1, ids, N, K, d, chunk, sums, counts);
}

/* Baseline scatter (_kernels.py:107-115): one merge per point, ascending. */
ORC_API void orc_scatter_f32(const float* X, const int32_t* ids, int64_t N, int64_t d, double* sums,
                             int64_t* counts) {
  for (int64_t i = 0; i < N; ++i) {
    double* dst = sums + (int64_t)ids[i] * d;
    for (int64_t j = 0; j < d; ++j) dst[j] += (double)X[i * d + j];
    counts[ids[i]] += 1;
  }
}

ORC_API void orc_scatter_f64(const double* X, const int32_t* ids, int64_t N, int64_t d,
                             double* sums, int64_t* counts) {
  for (int64_t i = 0; i < N; ++i) {
    double* dst = sums + (int64_t)ids[i] * d;
    for (int64_t j = 0; j < d; ++j) dst[j] += X[i * d + j];
    counts[ids[i]] += 1;
  }
}

/* ------------------------------------------------------------- normalize */
/* baseline.normalize (baseline.py:127-150): means = sums/counts in f64, cast
 * to the data dtype; empty clusters keep the previous row bitwise.
 * empty[k] = 1 for empty clusters. */
ORC_API void orc_normalize_f32(const double* sums, const int64_t* counts, const float* prev,
                               int64_t K, int64_t d, float* out, uint8_t* empty) {
  for (int64_t k = 0; k < K; ++k) {
    if (counts[k] > 0) {
      for (int64_t j = 0; j < d; ++j)
        out[k * d + j] = (float)(sums[k * d + j] / (double)counts[k]);
      empty[k] = 0;
    } else {
      memcpy(out + k * d, prev + k * d, sizeof(float) * (size_t)d);
      empty[k] = 1;
    }
  }
}

ORC_API void orc_normalize_f64(const double* sums, const int64_t* counts, const double* prev,
                               int64_t K, int64_t d, double* out, uint8_t* empty) {
  for (int64_t k = 0; k < K; ++k) {
    if (counts[k] > 0) {
      for (int64_t j = 0; j < d; ++j) out[k * d + j] = sums[k * d + j] / (double)counts[k];
      empty[k] = 0;
    } else {
      memcpy(out + k * d, prev + k * d, sizeof(double) * (size_t)d);
      empty[k] = 1;
    }
  }
}

/* ------------------------------------------------------------- k-means++
 * _kmeanspp_indices (core.py:342-357) leans on three numpy operations whose
 * arithmetic is restated here (numpy 2.3.5, the reference's own dependency):
 *   np.square(p64 - c).sum(axis=1) and min_d2.sum(): numpy's pairwise_sum
 *     (numpy/_core/src/umath/loops_utils.h.src, PW_BLOCKSIZE = 128): n < 8
 *     sequential from 0.0; n <= 128 eight strided accumulators combined as
 *     ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail; above 128
 *     split at n2 = n/2 - (n/2)%8 and add the halves;
 *   rng.choice(n, p=min_d2/total): cdf = cumsum(p) (serial), cdf /= cdf[-1],
 *     searchsorted(cdf, u, side="right") with u = rng.random().
 * The bitwise agreement with numpy is pinned by tests/test_oracle_golden.py. */
static double orc_pw(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] += a[i + k];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return orc_pw(a, n2) + orc_pw(a + n2, n - n2);
}

ORC_API double orc_pairwise_sum(const double* a, int64_t n) { return orc_pw(a, n); }

/* min_d2 = (first ? d2 : min(min_d2, d2)), d2_i = pairwise sum_j (x_ij - c_j)^2
 * over the f64 points (the reference upcasts with astype(float64)). */
ORC_API void orc_kmeanspp_sweep(const double* x, int64_t n, int64_t d, const double* c,
                                double* m, int first) {
#pragma omp parallel
  {
    double* sq = (double*)malloc(sizeof(double) * (size_t)d);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      const double* r = x + i * d;
      for (int64_t j = 0; j < d; ++j) {
        const double t = r[j] - c[j];
        sq[j] = t * t;
      }
      const double v = orc_pw(sq, d);
      if (first || v < m[i]) m[i] = v;
    }
    free(sq);
  }
}

/* searchsorted(cumsum(m / total) / cumsum[-1], u, side="right"). */
ORC_API int64_t orc_choice_cdf(const double* m, int64_t n, double total, double u) {
  double* cdf = (double*)malloc(sizeof(double) * (size_t)n);
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    s += m[i] / total;
    cdf[i] = s;
  }
  const double last = cdf[n - 1];
  int64_t lo = 0, hi = n; /* first index with cdf/last > u */
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (cdf[mid] / last > u)
      hi = mid;
    else
      lo = mid + 1;
  }
  free(cdf);
  return lo;
}
