// fk_assign_split.cu -- FlashAssign for f32 / f64 data on the tensor cores,
// bitwise equal to the reference's dot_mode="exact" (certified argmin).
//
// Replaces flash_assign (reference flash_assign.py:135-222) for the
// reference's own precisions.  The exact arithmetic (SURVEY Appendix A,
// _kernels.py:32-45) is a scalar f64 chain per (point, centroid); running it
// for all N*K pairs is FP64-add bound.  Instead:
//
//  1. split: every value v becomes two bf16 terms hi = bf16(v),
//     lo = bf16(v - hi), |v - hi - lo| <= 2^-16 |v|.  X2 / C2 rows are
//     [hi (16 ns) | lo (16 ns)], ns = ceil(d / 16) K=16 steps.
//  2. the tcgen05 pair kernel (fk_assign_tc.cu, SPLIT) accumulates
//     hi.hi + hi.lo + lo.hi (3 ns MMAs) plus the ||c||^2/2 bias step in fp32
//     TMEM and returns per row the estimated argmin a~, its score s~ and a
//     lower bound s2 on every other centroid's score.
//  3. certify (k_certify): with E = |s~ - s| bounded by the split and
//     accumulation errors and R by the reference's own roundings,
//     s2 - s~ > margin >= 2E + R proves a~ is the unique minimiser of the
//     reference's rounded distances, so a~ IS the reference's answer; its
//     distance is then recomputed with the reference arithmetic (bitwise).
//     The bound used (s units):
//        margin = 2^-11 (|x| cmax + cmax^2) + 2^-18 ||x||^2 + 2^-100
//     against the worst case 2E + R <= 2^-12.3 (|x| cmax + cmax^2/2) +
//     2^-19 (||x||^2 + cmax^2 + |x| cmax): split 3 * 2^-16 per product,
//     fp32 accumulation with truncation <= 17 * 2^-23 per K=16 MMA over
//     3 ns + 1 MMAs (d <= 128), f32 storage of the scores.
//  4. rows that fail (near-ties, exact ties, duplicates, non-finite or
//     near-underflow data, ids < 0) run the exact CUDA-core mirror over all
//     K centroids (fk_assign_exact.cu, row-list variant).
//
// dot_mode="fast" (the reference's relaxed mode, _kernels.py:85-104) runs the
// same certified path (fk_api.cu): it is exact.  k_certify's `fast` switch
// (keep every valid estimate) exists for measurements of the fallback's cost.
#include "fk_common.cuh"
#include "fk_kernels.h"

namespace fk {

FK_DEV __nv_bfloat16 to_bf16_rn(float v) { return __float2bfloat16_rn(v); }
FK_DEV __nv_bfloat16 to_bf16_rn(double v) { return __double2bfloat16(v); }

// --------------------------------------------------------------- split rows
// (rows, d) -> (rows, 32 ns) bf16 [hi | lo], zero padded to 16 ns each half.
// Two elements per thread: 4-byte bf16x2 stores.
template <typename T>
__global__ void __launch_bounds__(256)
    k_split_rows(const T* __restrict__ M, int64_t rows, int d, int dp, __nv_bfloat16* __restrict__ out) {
  const int hp = dp >> 1;  // element pairs per half row
  const int64_t total = rows * hp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / hp;
    const int j = 2 * (int)(i - r * hp);
    const T* src = M + r * d;
    const T v0 = j < d ? src[j] : (T)0;
    const T v1 = j + 1 < d ? src[j + 1] : (T)0;
    const __nv_bfloat16 h0 = to_bf16_rn(v0), h1 = to_bf16_rn(v1);
    const __nv_bfloat16 l0 = to_bf16_rn(v0 - (T)__bfloat162float(h0));
    const __nv_bfloat16 l1 = to_bf16_rn(v1 - (T)__bfloat162float(h1));
    __nv_bfloat162* row = reinterpret_cast<__nv_bfloat162*>(out + r * (2 * (int64_t)dp));
    row[j >> 1] = __halves2bfloat162(h0, h1);
    row[hp + (j >> 1)] = __halves2bfloat162(l0, l1);
  }
}

// ---------------------------------------------------------- split centroids
// One warp per padded centroid row: the [hi | lo] operand row, the bias
// operand [hi, mid, lo] of ||c||^2/2 (+inf beyond K) and cmax[b] = an upper
// bound on max_k ||c_k|| (float bits, atomicMax; pre-zeroed).
template <typename T>
__global__ void __launch_bounds__(256)
    k_split_centroids(const T* __restrict__ C, int64_t B, int64_t K, int d, int dp, int kpad,
                      __nv_bfloat16* __restrict__ c2, __nv_bfloat16* __restrict__ ext,
                      unsigned int* __restrict__ cmax, T* __restrict__ ct) {
  const int64_t gi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gi >= B * kpad) return;
  const int64_t b = gi / kpad, k = gi - b * kpad;
  __nv_bfloat16* o = ext + gi * 16;
  if (k >= K) {
    if (lane < 16)
      o[lane] = lane == 0 ? __float2bfloat16(__int_as_float(0x7f800000)) : __float2bfloat16(0.f);
    return;
  }
  const T* p = C + (b * K + k) * d;
  __nv_bfloat16* q = c2 + (b * K + k) * (2 * (int64_t)dp);
  double acc = 0.0;
  for (int j = lane; j < dp; j += 32) {
    const T v = j < d ? p[j] : (T)0;
    const __nv_bfloat16 h = to_bf16_rn(v);
    if (j < d) ct[(b * d + j) * K + k] = v;  // (B, d, K): coalesced centroid columns
    q[j] = h;
    q[dp + j] = to_bf16_rn(v - (T)__bfloat162float(h));
    acc = fma((double)v, (double)v, acc);
  }
  for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  const double v = 0.5 * acc;
  const __nv_bfloat16 hi = to_bf16_rn(v);
  const double r1 = v - (double)__bfloat162float(hi);
  const __nv_bfloat16 mid = to_bf16_rn(r1);
  const __nv_bfloat16 lo = to_bf16_rn(r1 - (double)__bfloat162float(mid));
  if (lane < 16) o[lane] = lane == 0 ? hi : lane == 1 ? mid : lane == 2 ? lo : __float2bfloat16(0.f);
  if (lane == 0) {
    // sqrt rounded up, then one more ulp of slack for the f64 sum's rounding
    float nrm = __double2float_ru(sqrt(acc));
    nrm = nrm * (1.0f + 0x1p-20f);
    if (!(nrm == nrm)) nrm = __int_as_float(0x7f800000);  // NaN -> +inf (never certifies)
    atomicMax(cmax + b, __float_as_uint(nrm));
  }
}

// the reference's product term fl64(fl_T(x * c)) (_kernels.py:39-41)
FK_DEV double prod_term(float x, float c) { return (double)__fmul_rn(x, c); }
FK_DEV double prod_term(double x, double c) { return __dmul_rn(x, c); }

// ---------------------------------------------------------------- certify
// One thread per row: the margin test (with the reference's ||x||^2, cached
// next to X's split operand), and for certified rows the reference distance to
// the chosen centroid.  Rows that do not certify go to the per-batch fallback list.
// The block's 128 rows and their chosen centroid rows stream through shared
// memory DC columns at a time (coalesced row reads, double-buffered: the next
// chunk's loads are in flight while the current one is summed); each thread
// runs its two serial f64 chains in ascending j, the reference's order.
template <typename T>
__global__ void __launch_bounds__(128)
    k_certify(const T* __restrict__ X, const T* __restrict__ C, const T* __restrict__ cn_ref,
              const unsigned int* __restrict__ cmax, int64_t N, int64_t K, int d,
              const int32_t* __restrict__ ids, const float* __restrict__ est,
              const float* __restrict__ second, const int8_t* __restrict__ stat,
              const T* __restrict__ xn_in, T* __restrict__ mind_out,
              const int32_t* __restrict__ idx_prev, int32_t* changed, int32_t* __restrict__ list,
              int32_t* __restrict__ list_cnt, int fast) {
  constexpr int DC = sizeof(T) == 4 ? 16 : 8;
  __shared__ T xs[2][DC][129];
  __shared__ T cs[2][DC][129];
  __shared__ int32_t sid[128];
  const int64_t b = blockIdx.y;
  const int64_t row0 = blockIdx.x * (int64_t)128;
  const int tid = threadIdx.x;
  const int64_t row = row0 + tid;
  const int64_t o = b * N + row;
  int32_t id = -1;
  if (row < N) id = ids[o];
  const bool valid = id >= 0 && id < K;
  sid[tid] = valid ? id : -1;
  __syncthreads();
  T px[DC], pc[DC];
  auto fetch = [&](int j0) {
#pragma unroll
    for (int i = 0; i < DC; ++i) {
      const int e = tid + 128 * i;
      const int r = e / DC, jj = e - r * DC;
      const int64_t gr = row0 + r;
      const int j = j0 + jj;
      const bool in = gr < N && j < d;
      const int32_t cid = sid[r];
      px[i] = in ? __ldg(X + (b * N + gr) * d + j) : (T)0;
      pc[i] = (in && cid >= 0) ? __ldg(C + (b * K + cid) * d + j) : (T)0;
    }
  };
  double da = 0.0;
  const int nch = (d + DC - 1) / DC;
  fetch(0);
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
#pragma unroll
    for (int i = 0; i < DC; ++i) {
      const int e = tid + 128 * i;
      const int r = e / DC, jj = e - r * DC;
      xs[buf][jj][r] = px[i];
      cs[buf][jj][r] = pc[i];
    }
    __syncthreads();
    if (c + 1 < nch) fetch((c + 1) * DC);
    const int jn = d - c * DC < DC ? d - c * DC : DC;
    for (int jj = 0; jj < jn; ++jj) {
      const T xv = xs[buf][jj][tid], cv = cs[buf][jj][tid];
      da = __dadd_rn(da, prod_term(xv, cv));
    }
  }
  bool flag = false, ch = false;
  // stat 1: the epilogue listed this row's candidate chunks (k_candidates)
  if (row < N && stat[o] != 1) {
    const T xn = xn_in[o];
    const double xa = (double)xn;
    const float cm = __uint_as_float(cmax[b]);
    const float nx = __fsqrt_ru(__double2float_ru(xa)) * (1.0f + 0x1p-20f);
    const float scale = __fmaf_ru(nx, cm, cm * cm);
    const float margin = 0x1p-11f * scale + 0x1p-18f * __double2float_ru(xa) + 0x1p-100f;
    const float gap = second[o] - est[o];
    // certified: a real gap wider than the margin (false for NaN / inf) and
    // operands well above the bf16 underflow range
    const bool cert = valid && (fast || (gap > margin && scale > 0x1p-60f && margin < 3e38f));
    if (cert) {
      T sv;
      if constexpr (sizeof(T) == 4) sv = __fadd_rn(xn, cn_ref[b * K + id]);
      else sv = __dadd_rn(xn, cn_ref[b * K + id]);
      double dv = __dsub_rn((double)sv, __dmul_rn(2.0, da));
      if (dv < 0.0) dv = 0.0;
      mind_out[o] = (T)dv;
      if (idx_prev) ch = idx_prev[o] != id;
    } else {
      flag = true;
    }
  }
  // warp-aggregated append to the fallback list (order is irrelevant: each
  // row's result depends on the row alone)
  const unsigned m = __ballot_sync(0xffffffffu, flag);
  if (m) {
    const int lane = tid & 31;
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(list_cnt + b, __popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (flag) list[b * N + base + __popc(m & ((1u << lane) - 1))] = (int32_t)row;
  }
  if (changed && __any_sync(0xffffffffu, ch) && (tid & 31) == 0) atomicOr(changed, 1);
}

// --------------------------------------------------------------- fallback
// The rows k_certify could not settle.  Two stages per row, both sweeping
// the centroids in tiles of 128 with the fp32 transposed C staged in shared
// memory (coalesced, shared by the block's FB_W * FB_R rows; lane = centroid
// owns 4 consecutive centroids of the tile, FB_R rows: 16 independent fp32
// chains fed by 16-byte shared-memory reads):
//  A. an fp32 FMA estimate D~_k = xn + cn_k - 2 sum_j x_j c_kj of every
//     distance and its row minimum dmin;
//  B. the same estimate again (bitwise the same values), and for every
//     centroid with NOT(D~_k > dmin + thr) the reference arithmetic
//     (fl64(fl_T(x c)) summed in ascending j, the exact mirror's formula).
// thr bounds 2 (E + R): E the estimate's error (fp32 rounding of the inputs,
// d+2 FMA roundings, the final adds), R the reference's own roundings, with a
// factor 4 of slack; the exact minimiser and every centroid tied with it are
// therefore candidates.  NaN / inf estimates are candidates.  Each lane scans
// its candidates in ascending id with strict '<' and the warp merge is
// lexicographic in (value, id): the lowest id among equal minima wins
// (rowmin_merge, _kernels.py:64-82).
constexpr int FB_W = 8, FB_R = 4, FB_KT = 128, FB_DC = 32;
template <typename T>
__global__ void __launch_bounds__(FB_W * 32)
    k_fallback_rows(const T* __restrict__ X, const T* __restrict__ C, const T* __restrict__ ct,
                    const T* __restrict__ cn, const T* __restrict__ xn_ref,
                    const unsigned int* __restrict__ cmax, int64_t B, int64_t N, int64_t K, int d,
                    const int32_t* __restrict__ list, const int32_t* __restrict__ list_cnt,
                    int32_t* __restrict__ idx_out, T* __restrict__ mind_out,
                    const int32_t* __restrict__ idx_prev, int32_t* changed) {
  constexpr int RB = FB_W * FB_R;  // rows per block
  __shared__ __align__(16) float cts[FB_DC][FB_KT];
  extern __shared__ __align__(16) uint8_t fb_sm[];
  float* xf = reinterpret_cast<float*>(fb_sm);  // (RB, d) fp32 copies of the rows
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int dp = (d + 3) & ~3;  // shared row stride: float4 reads
  bool ch = false;
  for (int64_t b = 0; b < B; ++b) {
    const int64_t cnt = list_cnt[b];
    const T* ctb = ct + b * d * K;
    const float cm = __uint_as_float(cmax[b]);
    for (int64_t i0 = (int64_t)blockIdx.x * RB; i0 < cnt; i0 += (int64_t)gridDim.x * RB) {
      int64_t o[FB_R];
      T xn[FB_R], best[FB_R];
      float xnf[FB_R], dmin[FB_R], thr[FB_R];
      int32_t bi[FB_R];
      __syncthreads();  // the previous rows' xf reads are done
#pragma unroll
      for (int q = 0; q < FB_R; ++q) {
        const int64_t i = i0 + wib * FB_R + q;
        const bool live = i < cnt;
        o[q] = live ? b * N + list[b * N + i] : -1;
        for (int j = lane; j < dp; j += 32)
          xf[(wib * FB_R + q) * dp + j] = (live && j < d) ? (float)X[o[q] * d + j] : 0.f;
        xn[q] = live ? xn_ref[o[q]] : (T)0;
        xnf[q] = (float)xn[q];
        const float nx = sqrtf(xnf[q]) * (1.f + 0x1p-20f);
        // E <= 2^-22 (xn + cmax^2) + (d + 4) 2^-23 |x| cmax;  R <= 2^-20 (xn + cmax^2 + |x| cmax)
        const float e = 0x1p-22f * (xnf[q] + cm * cm) + (float)(d + 4) * 0x1p-23f * nx * cm;
        const float r = 0x1p-20f * (xnf[q] + cm * cm + nx * cm);
        thr[q] = 8.f * (e + r);  // 2 (E + R) with a factor 4 of slack
        dmin[q] = __int_as_float(0x7f800000);
        best[q] = (T)__int_as_float(0x7f800000);
        bi[q] = -1;
      }
      const float* xw = xf + (int64_t)wib * FB_R * dp;
      for (int stage = 0; stage < 2; ++stage) {
        for (int64_t kb = 0; kb < K; kb += FB_KT) {
          float acc[FB_R][4];
#pragma unroll
          for (int q = 0; q < FB_R; ++q)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[q][u] = 0.f;
          for (int j0 = 0; j0 < d; j0 += FB_DC) {
            __syncthreads();
#pragma unroll
            for (int e = threadIdx.x; e < FB_DC * FB_KT; e += FB_W * 32) {
              const int jj = e / FB_KT, kk = e - jj * FB_KT;
              const int j = j0 + jj;
              const int64_t k = kb + kk;
              cts[jj][kk] = (j < d && k < K) ? (float)__ldg(ctb + (int64_t)j * K + k) : 0.f;
            }
            __syncthreads();
            const int jn = d - j0 < FB_DC ? d - j0 : FB_DC;
            for (int jj = 0; jj < jn; jj += 4) {  // rows are zero padded to a multiple of 4
              float4 xv[FB_R];
#pragma unroll
              for (int q = 0; q < FB_R; ++q)
                xv[q] = *reinterpret_cast<const float4*>(xw + q * dp + j0 + jj);
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float4 c4 = *reinterpret_cast<const float4*>(&cts[jj + t][4 * lane]);
#pragma unroll
                for (int q = 0; q < FB_R; ++q) {
                  const float x1 = t == 0 ? xv[q].x : t == 1 ? xv[q].y : t == 2 ? xv[q].z : xv[q].w;
                  acc[q][0] = fmaf(x1, c4.x, acc[q][0]);
                  acc[q][1] = fmaf(x1, c4.y, acc[q][1]);
                  acc[q][2] = fmaf(x1, c4.z, acc[q][2]);
                  acc[q][3] = fmaf(x1, c4.w, acc[q][3]);
                }
              }
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t k = kb + 4 * lane + u;  // the lane's 4 consecutive centroids, ascending
            if (k < K) {
              const T cnk = cn[b * K + k];
#pragma unroll
              for (int q = 0; q < FB_R; ++q) {
                const float dt = (xnf[q] + (float)cnk) - 2.f * acc[q][u];
                if (stage == 0) {
                  dmin[q] = fminf(dmin[q], dt);
                } else if (o[q] >= 0 && !(dt > dmin[q] + thr[q])) {
                  // candidate: the reference distance, ascending j
                  const T* xr = X + o[q] * d;
                  const T* cr = C + (b * K + k) * d;
                  double da = 0.0;
                  for (int j = 0; j < d; ++j) da = __dadd_rn(da, prod_term(xr[j], cr[j]));
                  T sv;
                  if constexpr (sizeof(T) == 4) sv = __fadd_rn(xn[q], cnk);
                  else sv = __dadd_rn(xn[q], cnk);
                  double dv = __dsub_rn((double)sv, __dmul_rn(2.0, da));
                  if (dv < 0.0) dv = 0.0;
                  const T v = (T)dv;
                  if (v < best[q]) {
                    best[q] = v;
                    bi[q] = (int32_t)k;
                  }
                }
              }
            }
          }
        }
        if (stage == 0) {
#pragma unroll
          for (int q = 0; q < FB_R; ++q)
#pragma unroll
            for (int sh = 16; sh; sh >>= 1)
              dmin[q] = fminf(dmin[q], __shfl_xor_sync(0xffffffffu, dmin[q], sh));
        }
      }
#pragma unroll
      for (int q = 0; q < FB_R; ++q) {
#pragma unroll
        for (int sh = 16; sh; sh >>= 1) {
          const T ob = __shfl_xor_sync(0xffffffffu, best[q], sh);
          const int32_t oi = __shfl_xor_sync(0xffffffffu, bi[q], sh);
          if (ob < best[q] || (ob == best[q] && oi >= 0 && (bi[q] < 0 || oi < bi[q]))) {
            best[q] = ob;
            bi[q] = oi;
          }
        }
        if (o[q] >= 0 && lane == 0) {
          idx_out[o[q]] = bi[q];
          mind_out[o[q]] = best[q];
          if (idx_prev && idx_prev[o[q]] != bi[q]) ch = true;
        }
      }
    }
  }
  if (changed && __any_sync(0xffffffffu, ch) && lane == 0) atomicOr(changed, 1);
}

// -------------------------------------------------------------- candidates
// Rows the epilogue could not certify but whose near chunks it listed: the
// exact argmin is in one of those <= 8 chunks of 32 centroids (a chunk is
// listed when its estimated minimum came within the certificate margin of the
// running best).  One warp per record:
//  1. an fp32 FMA estimate of every listed centroid's distance (lane =
//     centroid of the chunk, coalesced reads of the transposed C), with the
//     fallback's rigorous bound thr >= 2 (E + R);
//  2. the centroids with NOT(D~ > min D~ + thr) -- the exact minimiser and
//     everything tied with it -- compacted and evaluated with the reference
//     arithmetic, lanes = candidates; lexicographic (value, id) selection.
template <typename T>
__global__ void __launch_bounds__(256)
    k_candidates(const T* __restrict__ X, const T* __restrict__ ct, const T* __restrict__ cn,
                 const T* __restrict__ xn_ref, const unsigned int* __restrict__ cmax, int64_t N,
                 int64_t K, int d, const int32_t* __restrict__ rec,
                 const int32_t* __restrict__ rec_cnt, int rec_cap, int32_t* __restrict__ idx_out,
                 T* __restrict__ mind_out, const int32_t* __restrict__ idx_prev, int32_t* changed) {
  constexpr int NQ = kSplitRecInts - 2;  // chunks per record (max)
  extern __shared__ __align__(16) uint8_t cd_sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  T* xs = reinterpret_cast<T*>(cd_sm) + (int64_t)wib * d;
  __shared__ int32_t cand[8][NQ * 32];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t cnt = *rec_cnt < rec_cap ? *rec_cnt : rec_cap;
  bool ch = false;
  for (int64_t i = gw; i < cnt; i += nw) {
    const int32_t* r = rec + i * kSplitRecInts;
    const int64_t o = r[0];
    const int64_t b = o / N;
    const int n = r[1];
    __syncwarp();
    for (int j = lane; j < d; j += 32) xs[j] = X[o * d + j];
    __syncwarp();
    const T xn = xn_ref[o];
    const T* ctb = ct + b * d * K;
    const float cm = __uint_as_float(cmax[b]);
    const float xnf = (float)xn;
    const float nx = sqrtf(xnf) * (1.f + 0x1p-20f);
    const float e = 0x1p-22f * (xnf + cm * cm) + (float)(d + 4) * 0x1p-23f * nx * cm;
    const float rr = 0x1p-20f * (xnf + cm * cm + nx * cm);
    const float thr = 8.f * (e + rr);  // 2 (E + R) with a factor 4 of slack (as k_fallback_rows)
    // 1. fp32 estimates
    float dt[NQ];
    float dmin = __int_as_float(0x7f800000);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      dt[q] = __int_as_float(0x7f800000);
      if (q < n) {
        const int64_t k = (int64_t)r[2 + q] + lane;
        if (k < K) {
          const T* col = ctb + k;
          float acc = 0.f;
#pragma unroll 8
          for (int j = 0; j < d; ++j) acc = fmaf((float)xs[j], (float)__ldg(col + (int64_t)j * K), acc);
          dt[q] = (xnf + (float)cn[b * K + k]) - 2.f * acc;
          dmin = fminf(dmin, dt[q]);
        }
      }
    }
#pragma unroll
    for (int sh = 16; sh; sh >>= 1) dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, sh));
    // 2. compact the candidates (NaN / inf estimates included), then exact
    int nc = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (q < n) {
        const int64_t k = (int64_t)r[2 + q] + lane;
        const bool c = k < K && !(dt[q] > dmin + thr);
        const unsigned m = __ballot_sync(0xffffffffu, c);
        if (c) cand[wib][nc + __popc(m & ((1u << lane) - 1))] = (int32_t)k;
        nc += __popc(m);
      }
    }
    __syncwarp();
    T best = (T)__int_as_float(0x7f800000);
    int32_t bi = -1;
    for (int c0 = 0; c0 < nc; c0 += 32) {
      if (c0 + lane < nc) {
        const int64_t k = cand[wib][c0 + lane];
        const T* col = ctb + k;
        double da = 0.0;
        for (int j = 0; j < d; ++j) da = __dadd_rn(da, prod_term(xs[j], __ldg(col + (int64_t)j * K)));
        T sv;
        if constexpr (sizeof(T) == 4) sv = __fadd_rn(xn, cn[b * K + k]);
        else sv = __dadd_rn(xn, cn[b * K + k]);
        double dv = __dsub_rn((double)sv, __dmul_rn(2.0, da));
        if (dv < 0.0) dv = 0.0;
        const T v = (T)dv;
        if (v < best || (v == best && (bi < 0 || k < bi))) {
          best = v;
          bi = (int32_t)k;
        }
      }
    }
#pragma unroll
    for (int sh = 16; sh; sh >>= 1) {
      const T ob = __shfl_xor_sync(0xffffffffu, best, sh);
      const int32_t oi = __shfl_xor_sync(0xffffffffu, bi, sh);
      if (ob < best || (ob == best && oi >= 0 && (bi < 0 || oi < bi))) {
        best = ob;
        bi = oi;
      }
    }
    if (lane == 0) {
      idx_out[o] = bi;
      mind_out[o] = best;
      if (idx_prev && idx_prev[o] != bi) ch = true;
    }
  }
  if (changed && __any_sync(0xffffffffu, ch) && lane == 0) atomicOr(changed, 1);
}

// ---------------------------------------------------------------- launchers
bool assign_split_supported(int64_t d) { return d >= 1 && d <= 128; }

int split_steps(int64_t d) { return (int)((d + 15) / 16); }

cudaError_t launch_split_rows(int dt, const void* M, int64_t rows, int64_t d, void* out,
                              int num_sms, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  const int dp = 16 * split_steps(d);
  const int64_t total = rows * (dp / 2);
  int64_t grid = (total + 255) / 256;
  if (grid > (int64_t)num_sms * 16) grid = (int64_t)num_sms * 16;
  if (dt == DT_F64)
    k_split_rows<double><<<(unsigned)grid, 256, 0, s>>>((const double*)M, rows, (int)d, dp,
                                                        (__nv_bfloat16*)out);
  else
    k_split_rows<float><<<(unsigned)grid, 256, 0, s>>>((const float*)M, rows, (int)d, dp,
                                                       (__nv_bfloat16*)out);
  return cudaGetLastError();
}

cudaError_t launch_split_centroids(int dt, const void* C, int64_t B, int64_t K, int64_t d,
                                   int kpad, void* c2, void* ext, unsigned int* cmax, void* ct,
                                   cudaStream_t s) {
  const int dp = 16 * split_steps(d);
  const int64_t n = B * kpad * 32;
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (dt == DT_F64)
    k_split_centroids<double><<<grid, 256, 0, s>>>((const double*)C, B, K, (int)d, dp, kpad,
                                                   (__nv_bfloat16*)c2, (__nv_bfloat16*)ext, cmax,
                                                   (double*)ct);
  else
    k_split_centroids<float><<<grid, 256, 0, s>>>((const float*)C, B, K, (int)d, dp, kpad,
                                                  (__nv_bfloat16*)c2, (__nv_bfloat16*)ext, cmax,
                                                  (float*)ct);
  return cudaGetLastError();
}

cudaError_t launch_certify(int dt, const void* X, const void* C, const void* cn_ref,
                           const unsigned int* cmax, int64_t B, int64_t N, int64_t K, int64_t d,
                           const int32_t* ids, const float* est, const float* second,
                           const int8_t* stat, const void* xn_in, void* mind_out,
                           const int32_t* idx_prev, int32_t* changed, int32_t* list,
                           int32_t* list_cnt, int fast, cudaStream_t s) {
  dim3 grid((unsigned)((N + 127) / 128), (unsigned)B);
  if (dt == DT_F64)
    k_certify<double><<<grid, 128, 0, s>>>((const double*)X, (const double*)C,
                                           (const double*)cn_ref, cmax, N, K, (int)d, ids, est,
                                           second, stat, (const double*)xn_in, (double*)mind_out,
                                           idx_prev, changed, list, list_cnt, fast);
  else
    k_certify<float><<<grid, 128, 0, s>>>((const float*)X, (const float*)C, (const float*)cn_ref,
                                          cmax, N, K, (int)d, ids, est, second, stat,
                                          (const float*)xn_in, (float*)mind_out, idx_prev, changed,
                                          list, list_cnt, fast);
  return cudaGetLastError();
}

cudaError_t launch_candidates(int dt, const void* X, const void* ct, const void* cn_ref,
                              const void* xn_ref, const unsigned int* cmax, int64_t N, int64_t K,
                              int64_t d,
                              const int32_t* rec, const int32_t* rec_cnt, int rec_cap,
                              int32_t* idx_out, void* mind_out, const int32_t* idx_prev,
                              int32_t* changed, int num_sms, cudaStream_t s) {
  const size_t smem = 8 * (size_t)d * (dt == DT_F64 ? 8 : 4);
  const unsigned grid = (unsigned)num_sms * 8;
  if (dt == DT_F64)
    k_candidates<double><<<grid, 256, smem, s>>>((const double*)X, (const double*)ct,
                                                 (const double*)cn_ref, (const double*)xn_ref, cmax, N, K,
                                                 (int)d, rec, rec_cnt, rec_cap, idx_out,
                                                 (double*)mind_out, idx_prev, changed);
  else
    k_candidates<float><<<grid, 256, smem, s>>>((const float*)X, (const float*)ct,
                                                (const float*)cn_ref, (const float*)xn_ref, cmax, N, K,
                                                (int)d, rec, rec_cnt, rec_cap, idx_out,
                                                (float*)mind_out, idx_prev, changed);
  return cudaGetLastError();
}

cudaError_t launch_fallback_rows(int dt, const void* X, const void* C, const void* ct,
                                 const void* cn, const void* xn_ref, const unsigned int* cmax,
                                 int64_t B, int64_t N, int64_t K, int64_t d, const int32_t* list,
                                 const int32_t* list_cnt, int32_t* idx_out, void* mind_out,
                                 const int32_t* idx_prev, int32_t* changed, int num_sms,
                                 cudaStream_t s) {
  const size_t smem = FB_W * FB_R * (size_t)((d + 3) & ~3) * 4;
  const unsigned grid = (unsigned)num_sms * 4;
  if (dt == DT_F64)
    k_fallback_rows<double><<<grid, FB_W * 32, smem, s>>>(
        (const double*)X, (const double*)C, (const double*)ct, (const double*)cn,
        (const double*)xn_ref, cmax, B, N, K, (int)d, list, list_cnt, idx_out, (double*)mind_out,
        idx_prev, changed);
  else
    k_fallback_rows<float><<<grid, FB_W * 32, smem, s>>>(
        (const float*)X, (const float*)C, (const float*)ct, (const float*)cn, (const float*)xn_ref,
        cmax, B, N, K, (int)d, list, list_cnt, idx_out, (float*)mind_out, idx_prev, changed);
  return cudaGetLastError();
}

FK_MODULE_ANCHOR(assign_split)

}  // namespace fk
