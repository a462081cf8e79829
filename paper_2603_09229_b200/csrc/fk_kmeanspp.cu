// fk_kmeanspp.cu -- k-means++ D^2 seeding on the device, index-for-index equal to
// the reference's numpy seeding (_kmeanspp_indices, core.py:342-357; the
// streamed variant _streaming_kmeanspp, pipeline.py:420-453).
//
// One draw j (1 <= j < K) of the reference is
//     min_d2 = min(min_d2, np.square(p64 - p64[idx[j-1]]).sum(axis=1))
//     total  = float(min_d2.sum())
//     idx[j] = rng.choice(n, p=min_d2 / total)  if total > 0 else rng.integers(n)
// and numpy's choice(n, p) is: cdf = cumsum(p); cdf /= cdf[-1];
// searchsorted(cdf, rng.random(), side="right").  The RNG stays on the host:
// the caller passes the doubles rng.random() returns (u) and idx[:, 0].
//
// Bitwise reproduction on the device:
//  * every row distance follows numpy's pairwise summation over d (8
//    accumulators for n <= 128, recursive halving at multiples of 8 above),
//    with separately rounded f64 subtract / square / add (no FMA contraction);
//  * `total` follows numpy's pairwise summation over the whole (N,) table:
//    the recursion tree is cut at the depth t1 where nodes hold <= 4096 rows;
//    one CTA reduces each node (k_pp_node), k_pp_tier folds the complete
//    binary tree above t1 -- the same additions in the same tree order;
//  * the sequential cumsum of p = min_d2/total is the one step that is
//    inherently serial.  k_pp_select finds the candidate index from an
//    exact (double-double) prefix of min_d2 and CERTIFIES it with a rigorous
//    bound on how far numpy's rounded cumsum/normalisation can be from the
//    exact prefix ratio (|cdf_i - r_i| <= D(i, r_i), derivation in DESIGN.md);
//    only when u falls inside that window (probability ~ N^2 * 2^-54, i.e.
//    ~0.4% of draws at N = 8M and ~1e-8 at N = 16k) k_pp_exact replays
//    numpy's serial cumsum + division + searchsorted literally.
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "fk_common.cuh"
#include "fk_kernels.h"

namespace fk {
namespace {

constexpr int kLeaf = 128;       // numpy PW_BLOCKSIZE (loops_utils.h.src)
constexpr int kNodeMax = 4096;   // rows per bottom node of the pairwise tree
constexpr int kTierLevels = 12;  // levels folded per k_pp_tier CTA (4096 inputs)
constexpr int kNodeLevels = 9;  // max relative depth inside a bottom node
constexpr int kSweepRows = 128;  // rows per sweep CTA (one row per thread)
constexpr int kExactTile = 2048; // fallback: p values staged per tile

__host__ __device__ inline int64_t pw_split(int64_t n) {
  const int64_t h = n >> 1;
  return h - (h & 7);
}

// Range of the node reached from the root (0, N) by `depth` decisions, path
// bits most significant first (0 = left half).
__host__ __device__ inline void pw_walk(int64_t N, int depth, int64_t path, int64_t& lo,
                                        int64_t& n) {
  lo = 0;
  n = N;
  for (int t = depth - 1; t >= 0; --t) {
    const int64_t h = pw_split(n);
    if ((path >> t) & 1) {
      lo += h;
      n -= h;
    } else {
      n = h;
    }
  }
}

FK_DEV int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }

FK_DEV double to_f64(float v) { return (double)v; }
FK_DEV double to_f64(double v) { return v; }
FK_DEV double to_f64(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
FK_DEV double to_f64(__half v) { return (double)__half2float(v); }

// 8 consecutive elements (16-byte aligned) widened to f64.
template <typename T>
FK_DEV void load8(const T* p, double* o);
// bf16 -> f32 is a 16-bit shift (exact); f32 -> f64 one F2F.
template <>
FK_DEV void load8<__nv_bfloat16>(const __nv_bfloat16* p, double* o) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    o[2 * k] = (double)__uint_as_float(w[k] << 16);
    o[2 * k + 1] = (double)__uint_as_float(w[k] & 0xffff0000u);
  }
}
template <>
FK_DEV void load8<__half>(const __half* p, double* o) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const __half2 h = *reinterpret_cast<const __half2*>(&w[k]);
    const float2 f = __half22float2(h);
    o[2 * k] = (double)f.x;
    o[2 * k + 1] = (double)f.y;
  }
}
template <>
FK_DEV void load8<float>(const float* p, double* o) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 4);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
template <>
FK_DEV void load8<double>(const double* p, double* o) {
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const double2 v = *reinterpret_cast<const double2*>(p + k);
    o[k] = v.x;
    o[k + 1] = v.y;
  }
}

FK_DEV double sqd(double x, double c) {
  const double t = __dsub_rn(x, c);
  return __dmul_rn(t, t);
}

// numpy pairwise_sum leaf (n <= 128) of (x_k - c_k)^2, x a 16-B aligned row.
template <typename T>
FK_DEV double pw_leaf_row(const T* x, const double* c, int n) {
  if (n < 8) {
    double res = 0.;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, sqd(to_f64(x[i]), c[i]));
    return res;
  }
  double r[8], v[8];
  load8<T>(x, v);
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = sqd(v[k], c[k]);
  int i = 8;
  const int body = n - (n % 8);
  for (; i < body; i += 8) {
    load8<T>(x + i, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], sqd(v[k], c[i + k]));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, sqd(to_f64(x[i]), c[i]));
  return res;
}

// Same leaf for a compile-time d (multiple of 8, 8 <= D <= 128): fully
// unrolled, centre read as 16-B pairs, no tail.
template <typename T, int D>
FK_DEV double pw_leaf_row_fixed(const T* x, const double* c) {
  static_assert(D % 8 == 0 && D >= 8 && D <= kLeaf, "fixed leaf");
  double r[8], v[8];
#pragma unroll
  for (int i = 0; i < D; i += 8) {
    load8<T>(x + i, v);
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      const double2 cc = *reinterpret_cast<const double2*>(c + i + k);
      const double s0 = sqd(v[k], cc.x), s1 = sqd(v[k + 1], cc.y);
      r[k] = i == 0 ? s0 : __dadd_rn(r[k], s0);
      r[k + 1] = i == 0 ? s1 : __dadd_rn(r[k + 1], s1);
    }
  }
  return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
}

// Compile-time d above 128: numpy's split into two halves of fixed size.
template <typename T, int D>
FK_DEV double pw_row_fixed(const T* x, const double* c) {
  if constexpr (D <= kLeaf) {
    return pw_leaf_row_fixed<T, D>(x, c);
  } else {
    constexpr int D2 = (D / 2) - (D / 2) % 8;
    const double a = pw_row_fixed<T, D2>(x, c);
    const double b = pw_row_fixed<T, D - D2>(x + D2, c + D2);
    return __dadd_rn(a, b);
  }
}

// Rows longer than 128: numpy splits at n2 = n/2 rounded down to a multiple of
// 8 (keeps every leaf 16-B aligned for all element types).
template <typename T>
__device__ __noinline__ double pw_row_rec(const T* x, const double* c, int n) {
  if (n <= kLeaf) return pw_leaf_row<T>(x, c, n);
  const int n2 = (int)pw_split(n);
  const double a = pw_row_rec<T>(x, c, n2);
  const double b = pw_row_rec<T>(x + n2, c + n2, n - n2);
  return __dadd_rn(a, b);
}

template <typename T>
FK_DEV double pw_row(const T* x, const double* c, int n) {
  return n <= kLeaf ? pw_leaf_row<T>(x, c, n) : pw_row_rec<T>(x, c, n);
}

// ------------------------------------------------------------ double-double
struct DD {
  double hi, lo;
};
FK_DEV DD dd_add(DD a, DD b) {
  const double s = __dadd_rn(a.hi, b.hi);
  const double bb = __dsub_rn(s, a.hi);
  double e = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b.hi, bb));
  e = __dadd_rn(e, __dadd_rn(a.lo, b.lo));
  const double hi = __dadd_rn(s, e);
  return {hi, __dsub_rn(e, __dsub_rn(hi, s))};
}
FK_DEV DD dd_add1(DD a, double b) { return dd_add(a, DD{b, 0.0}); }
FK_DEV DD dd_mul1(DD a, double b) {  // (a.hi + a.lo) * b
  const double p = __dmul_rn(a.hi, b);
  double e = __fma_rn(a.hi, b, -p);
  e = __fma_rn(a.lo, b, e);
  const double hi = __dadd_rn(p, e);
  return {hi, __dsub_rn(e, __dsub_rn(hi, p))};
}
FK_DEV bool dd_gt(DD a, DD b) { return a.hi > b.hi || (a.hi == b.hi && a.lo > b.lo); }
FK_DEV bool dd_le(DD a, DD b) { return !dd_gt(a, b); }
FK_DEV DD dd_shfl_up(DD v, int k) {
  return {__shfl_up_sync(0xffffffffu, v.hi, k), __shfl_up_sync(0xffffffffu, v.lo, k)};
}
FK_DEV DD dd_shfl_xor(DD v, int k) {
  return {__shfl_xor_sync(0xffffffffu, v.hi, k), __shfl_xor_sync(0xffffffffu, v.lo, k)};
}

// Block-wide exclusive scan of one DD per thread (blockDim multiple of 32,
// <= 1024); returns the exclusive prefix, *total gets the block sum.
FK_DEV DD block_excl_scan(DD v, DD* warp_buf, DD* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  DD inc = v;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const DD o = dd_shfl_up(inc, k);
    if (lane >= k) inc = dd_add(o, inc);
  }
  if (lane == 31) warp_buf[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    DD w = lane < nw ? warp_buf[lane] : DD{0.0, 0.0};
    DD wi = w;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const DD o = dd_shfl_up(wi, k);
      if (lane >= k) wi = dd_add(o, wi);
    }
    if (lane < nw) warp_buf[lane] = DD{wi.hi, wi.lo};  // inclusive over warps
  }
  __syncthreads();
  const DD wbase = warp > 0 ? warp_buf[warp - 1] : DD{0.0, 0.0};
  *total = warp_buf[nw - 1];
  const DD up = dd_shfl_up(inc, 1);  // all lanes take part in the shuffle
  return lane > 0 ? dd_add(wbase, up) : wbase;
}

// ------------------------------------------------------------------ sweep
// min_d2[b, i] = (first ? d2 : min(min_d2[b, i], d2)), d2 = numpy-order
// ||x_i - center_b||^2 in f64.  center_b = cen + b*cen_sb + (idx ? idx[b*K + col] : 0)*d.
template <typename T, int D>
__global__ void __launch_bounds__(kSweepRows) k_pp_sweep(
    const T* __restrict__ X, int64_t rows, int d, int64_t x_sb, const T* __restrict__ cen,
    int64_t cen_sb, const int64_t* __restrict__ idx, int64_t K, int64_t col,
    double* __restrict__ m, int64_t m_sb, int first, const int32_t* __restrict__ halted,
    int64_t j, int stride_elems) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int b = blockIdx.y;
  if (halted && halted[b] <= j - 1) return;  // total was 0 at an earlier draw: table stays 0
  double* c = reinterpret_cast<double*>(sm);
  T* tile = reinterpret_cast<T*>(sm + (((size_t)d * 8 + 15) & ~size_t(15)));
  const T* crow = cen + b * cen_sb + (idx ? idx[b * K + col] : 0) * (int64_t)d;
  for (int k = threadIdx.x; k < d; k += blockDim.x) c[k] = to_f64(crow[k]);
  const int64_t r0 = (int64_t)blockIdx.x * kSweepRows;
  const int nr = (int)i64min(kSweepRows, rows - r0);
  const T* src = X + b * x_sb + r0 * d;
  const int rb = d * (int)sizeof(T);
  if ((rb & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int vpr = rb >> 4;
    const int nv = nr * vpr;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    // (row, vector) of v = tid + k*blockDim, advanced without divisions
    const int dr = kSweepRows / vpr, dq = kSweepRows - dr * vpr;
    int r = threadIdx.x / vpr, q = threadIdx.x - r * vpr;
    constexpr int kU = 8;
    for (int v0 = threadIdx.x; v0 < nv; v0 += kU * kSweepRows) {
      uint4 buf[kU];
      int rr[kU], qq[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int v = v0 + u * kSweepRows;
        rr[u] = r;
        qq[u] = q;
        if (v < nv) buf[u] = s4[v];
        q += dq;
        r += dr;
        if (q >= vpr) {
          q -= vpr;
          ++r;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (v0 + u * kSweepRows < nv)
          *reinterpret_cast<uint4*>(tile + (size_t)rr[u] * stride_elems + qq[u] * (16 / sizeof(T))) =
              buf[u];
    }
  } else {
    const int ne = nr * d;
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
      const int r = e / d, q = e - r * d;
      tile[(size_t)r * stride_elems + q] = src[e];
    }
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < nr) {
    const double v = D > 0 ? pw_row_fixed<T, (D > 0 ? D : 8)>(tile + (size_t)t * stride_elems, c)
                           : pw_row<T>(tile + (size_t)t * stride_elems, c, d);
    double* mp = m + b * m_sb + r0 + t;
    *mp = first ? v : fmin(*mp, v);
  }
}

FK_DEV void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
FK_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
FK_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Persistent, software-pipelined sweep (rows of d*size % 16 == 0 bytes, 16-B
// aligned): each CTA walks tiles of 128 rows with a STAGES-deep cp.async ring
// (padded rows: conflict-free 16-B reads), so HBM streaming overlaps the f64
// arithmetic of the previous tiles.
template <typename T, int STAGES, int D>
__global__ void __launch_bounds__(kSweepRows) k_pp_sweep_pipe(
    const T* __restrict__ X, int64_t rows, int d, int64_t x_sb, const T* __restrict__ cen,
    int64_t cen_sb, const int64_t* __restrict__ idx, int64_t K, int64_t col,
    double* __restrict__ m, int64_t m_sb, int first, const int32_t* __restrict__ halted,
    int64_t j, int stride_elems) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int b = blockIdx.y;
  if (halted && halted[b] <= j - 1) return;
  double* c = reinterpret_cast<double*>(sm);
  T* tiles = reinterpret_cast<T*>(sm + (((size_t)d * 8 + 15) & ~size_t(15)));
  const size_t tile_elems = (size_t)kSweepRows * stride_elems;
  const T* crow = cen + b * cen_sb + (idx ? idx[b * K + col] : 0) * (int64_t)d;
  for (int k = threadIdx.x; k < d; k += blockDim.x) c[k] = to_f64(crow[k]);
  const int64_t ntiles = (rows + kSweepRows - 1) / kSweepRows;
  const T* xb = X + b * x_sb;
  const int vpr = (d * (int)sizeof(T)) >> 4;
  const int dr = kSweepRows / vpr, dq = kSweepRows - dr * vpr;
  const int r_init = threadIdx.x / vpr, q_init = threadIdx.x - r_init * vpr;
  constexpr int kEl = 16 / sizeof(T);
  auto issue = [&](int64_t t, int slot) {
    if (t < ntiles) {
      const int64_t r0 = t * kSweepRows;
      const int nr = (int)i64min(kSweepRows, rows - r0);
      const int nv = nr * vpr;
      const uint4* s4 = reinterpret_cast<const uint4*>(xb + r0 * d);
      T* dst = tiles + slot * tile_elems;
      int r = r_init, q = q_init;
      for (int v = threadIdx.x; v < nv; v += kSweepRows) {
        cp_async16(dst + (size_t)r * stride_elems + q * kEl, s4 + v);
        q += dq;
        r += dr;
        if (q >= vpr) {
          q -= vpr;
          ++r;
        }
      }
    }
    cp_async_commit();
  };
  int64_t t = blockIdx.x;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) issue(t + (int64_t)s * gridDim.x, s);
  int slot = 0;
  for (; t < ntiles; t += gridDim.x) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();  // tile t landed for every thread; slot (slot-1) is free again
    issue(t + (int64_t)(STAGES - 1) * gridDim.x, (slot + STAGES - 1) % STAGES);
    const int64_t r0 = t * kSweepRows;
    const int nr = (int)i64min(kSweepRows, rows - r0);
    if ((int)threadIdx.x < nr) {
      const T* xr = tiles + slot * tile_elems + (size_t)threadIdx.x * stride_elems;
      const double v = D > 0 ? pw_row_fixed<T, (D > 0 ? D : 8)>(xr, c) : pw_row<T>(xr, c, d);
      double* mp = m + b * m_sb + r0 + threadIdx.x;
      *mp = first ? v : fmin(*mp, v);
    }
    slot = (slot + 1) % STAGES;
  }
  cp_async_wait<0>();
}

// ------------------------------------------------ pruned sweep (in-core)
// Exact pruning of the D^2 sweep: a row whose new distance provably cannot go
// below its current minimum keeps it without being read.  With near = the
// chosen center that realised m and D = ||c_new - c_near||, the triangle
// inequality gives ||x - c_new|| >= D - ||x - c_near||.  m is within a
// relative ~d*2^-53 of ||x - c_near||^2 and D of the exact distance, so with
// 1e-9 margins (d <= 2^20) L^2 (1 - 1e-9) > m guarantees the numpy-order
// rounded d2 >= m, i.e. min(m, d2) == m bit for bit.  Rows that are not pruned
// are staged and computed exactly as in k_pp_sweep.
__global__ void __launch_bounds__(256) k_pp_cdist(const void* __restrict__ Xv, int dt, int64_t N,
                                                   int d, const int64_t* __restrict__ idx,
                                                   int64_t K, int64_t jc,
                                                   double* __restrict__ centers,
                                                   double* __restrict__ cdist,
                                                   const int32_t* __restrict__ halted, int64_t j) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int b = blockIdx.y;
  if (halted[b] <= j - 1) return;
  double* c = reinterpret_cast<double*>(sm);
  const int64_t row = idx[b * K + jc];
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    const int64_t e = (b * N + row) * (int64_t)d + k;
    double v;
    switch (dt) {
      case DT_F32: v = (double)static_cast<const float*>(Xv)[e]; break;
      case DT_F64: v = static_cast<const double*>(Xv)[e]; break;
      case DT_BF16: v = to_f64(static_cast<const __nv_bfloat16*>(Xv)[e]); break;
      default: v = to_f64(static_cast<const __half*>(Xv)[e]); break;
    }
    c[k] = v;
  }
  __syncthreads();
  double* cb = centers + (int64_t)b * K * d;
  if (blockIdx.x == 0)
    for (int k = threadIdx.x; k < d; k += blockDim.x) cb[jc * d + k] = c[k];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= jc) return;
  double acc = 0.0;
  for (int k = lane; k < d; k += 32) {
    const double t = cb[i * d + k] - c[k];
    acc += t * t;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) cdist[b * K + i] = sqrt(acc);
}

template <typename T, int D>
__global__ void __launch_bounds__(kSweepRows) k_pp_sweep_pruned(
    const T* __restrict__ X, int64_t N, int d, const int64_t* __restrict__ idx, int64_t K,
    int64_t col, double* __restrict__ m, int32_t* __restrict__ nearest,
    const double* __restrict__ cdist, int first, const int32_t* __restrict__ halted, int64_t j,
    int stride_elems) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int s_list[kSweepRows];
  __shared__ int s_wcnt[kSweepRows / 32];
  const int b = blockIdx.y;
  if (halted[b] <= j - 1) return;
  double* c = reinterpret_cast<double*>(sm);
  T* tile = reinterpret_cast<T*>(sm + (((size_t)d * 8 + 15) & ~size_t(15)));
  const T* xb = X + (int64_t)b * N * d;
  const T* crow = xb + idx[b * K + col] * (int64_t)d;
  for (int k = threadIdx.x; k < d; k += blockDim.x) c[k] = to_f64(crow[k]);
  const int64_t r0 = (int64_t)blockIdx.x * kSweepRows;
  const int nr = (int)i64min(kSweepRows, N - r0);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double* mb = m + (int64_t)b * N + r0;
  int32_t* nb = nearest + (int64_t)b * N + r0;
  bool need = false;
  double mm = 0.0;
  if (t < nr) {
    if (first) {
      need = true;
    } else {
      mm = mb[t];
      const double Dn = cdist[b * K + nb[t]];
      const double L = Dn * (1.0 - 1e-9) - sqrt(mm) * (1.0 + 1e-9);
      need = !(L > 0.0 && L * L * (1.0 - 1e-9) > mm);
    }
  }
  // compact the rows that must be computed
  const unsigned bal = __ballot_sync(0xffffffffu, need);
  if (lane == 0) s_wcnt[warp] = __popc(bal);
  __syncthreads();
  int base = 0, nneed = 0;
#pragma unroll
  for (int w = 0; w < kSweepRows / 32; ++w) {
    if (w < warp) base += s_wcnt[w];
    nneed += s_wcnt[w];
  }
  if (need) s_list[base + __popc(bal & ((1u << lane) - 1))] = t;
  __syncthreads();
  if (nneed == 0) return;
  // stage the needed rows (16-byte vectors, coalesced within each row)
  const int vpr = (d * (int)sizeof(T)) >> 4;
  constexpr int kEl = 16 / sizeof(T);
  const int nv = nneed * vpr;
  {
    // (slot, vector) of v = tid + k*blockDim advanced without divisions; 8 loads in flight
    const int dr = kSweepRows / vpr, dq = kSweepRows - dr * vpr;
    int sl = threadIdx.x / vpr, q = threadIdx.x - sl * vpr;
    constexpr int kU = 8;
    for (int v0 = threadIdx.x; v0 < nv; v0 += kU * kSweepRows) {
      uint4 buf[kU];
      int ss[kU], qq[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        ss[u] = sl;
        qq[u] = q;
        if (v0 + u * kSweepRows < nv)
          buf[u] = reinterpret_cast<const uint4*>(xb + (r0 + s_list[sl]) * (int64_t)d)[q];
        q += dq;
        sl += dr;
        if (q >= vpr) {
          q -= vpr;
          ++sl;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (v0 + u * kSweepRows < nv)
          *reinterpret_cast<uint4*>(tile + (size_t)ss[u] * stride_elems + qq[u] * kEl) = buf[u];
    }
  }
  __syncthreads();
  if (t < nneed) {
    const int rr = s_list[t];
    const T* xr = tile + (size_t)t * stride_elems;
    const double v = D > 0 ? pw_row_fixed<T, (D > 0 ? D : 8)>(xr, c) : pw_row<T>(xr, c, d);
    if (first) {
      mb[rr] = v;
      nb[rr] = (int32_t)col;
    } else if (v < mb[rr]) {
      mb[rr] = v;
      nb[rr] = (int32_t)col;
    }
  }
}

// Rows that do not fit the shared-memory tile: the same arithmetic straight
// from global memory (one row per thread; rows 16-B aligned when d*size%16==0).
template <typename T>
__global__ void __launch_bounds__(128) k_pp_sweep_global(
    const T* __restrict__ X, int64_t rows, int d, int64_t x_sb, const T* __restrict__ cen,
    int64_t cen_sb, const int64_t* __restrict__ idx, int64_t K, int64_t col,
    double* __restrict__ m, int64_t m_sb, int first, const int32_t* __restrict__ halted,
    int64_t j) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int b = blockIdx.y;
  if (halted && halted[b] <= j - 1) return;
  double* c = reinterpret_cast<double*>(sm);
  const T* crow = cen + b * cen_sb + (idx ? idx[b * K + col] : 0) * (int64_t)d;
  for (int k = threadIdx.x; k < d; k += blockDim.x) c[k] = to_f64(crow[k]);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const double v = pw_row<T>(X + b * x_sb + i * d, c, d);
  double* mp = m + b * m_sb + i;
  *mp = first ? v : fmin(*mp, v);
}

// Unaligned rows (d * size % 16 != 0) and no tile: element-wise leaf.
template <typename T>
__device__ __noinline__ double pw_scalar(const T* x, const double* c, int n) {
  if (n > kLeaf) {
    const int n2 = (int)pw_split(n);
    // bounded depth (d <= 2^20): at most 13 levels; explicit recursion below
    return __dadd_rn(pw_scalar(x, c, n2), pw_scalar(x + n2, c + n2, n - n2));
  }
  if (n < 8) {
    double res = 0.;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, sqd(to_f64(x[i]), c[i]));
    return res;
  }
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = sqd(to_f64(x[k]), c[k]);
  int i = 8;
  const int body = n - (n % 8);
  for (; i < body; i += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], sqd(to_f64(x[i + k]), c[i + k]));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, sqd(to_f64(x[i]), c[i]));
  return res;
}

template <typename T>
__global__ void __launch_bounds__(128) k_pp_sweep_scalar(
    const T* __restrict__ X, int64_t rows, int d, int64_t x_sb, const T* __restrict__ cen,
    int64_t cen_sb, const int64_t* __restrict__ idx, int64_t K, int64_t col,
    double* __restrict__ m, int64_t m_sb, int first, const int32_t* __restrict__ halted,
    int64_t j) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int b = blockIdx.y;
  if (halted && halted[b] <= j - 1) return;
  double* c = reinterpret_cast<double*>(sm);
  const T* crow = cen + b * cen_sb + (idx ? idx[b * K + col] : 0) * (int64_t)d;
  for (int k = threadIdx.x; k < d; k += blockDim.x) c[k] = to_f64(crow[k]);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const double v = pw_scalar<T>(X + b * x_sb + i * d, c, d);
  double* mp = m + b * m_sb + i;
  *mp = first ? v : fmin(*mp, v);
}

// ------------------------------------------------- pairwise total: bottom
// One CTA per node at depth t1 (<= 4096 rows): numpy's pairwise sum of the
// node's range (level by level inside shared memory), plus an exact-ish
// double-double sum of the same range for the selection scan.
__global__ void __launch_bounds__(256) k_pp_node(const double* __restrict__ m, int64_t N,
                                                  int64_t m_sb, int t1, int rdepth,
                                                  const int32_t* __restrict__ halted, int64_t j,
                                                  double* __restrict__ vals,
                                                  double2* __restrict__ ddsum) {
  __shared__ double a[kNodeMax];
  __shared__ double V[(2 << kNodeLevels) - 1];
  __shared__ uint8_t kind[(2 << kNodeLevels) - 1];
  __shared__ int leaf_lo[kNodeMax / 32], leaf_n[kNodeMax / 32], leaf_v[kNodeMax / 32];
  __shared__ int nleaf;
  __shared__ DD wb[32];
  const int b = blockIdx.y;
  if (halted && halted[b] < j) return;
  const int64_t node = blockIdx.x;
  int64_t lo0, n0;
  pw_walk(N, t1, node, lo0, n0);
  const double* src = m + b * m_sb + lo0;
  if (threadIdx.x == 0) nleaf = 0;
  DD acc{0.0, 0.0};
  for (int k = threadIdx.x; k < n0; k += blockDim.x) {
    const double v = src[k];
    a[k] = v;
    acc = dd_add1(acc, v);
  }
  // block reduction of the DD partial sums
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) acc = dd_add(acc, dd_shfl_xor(acc, k));
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    DD s{0.0, 0.0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = dd_add(s, wb[w]);
    ddsum[b * ((int64_t)1 << t1) + node] = make_double2(s.hi, s.lo);
  }
  // A: classify every node of the subtree (0 absent, 1 leaf, 2 internal), list the leaves
  for (int r = 0; r <= rdepth; ++r) {
    const int cnt = 1 << r;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
      int64_t lo = 0, n = n0;
      bool exists = true;
      for (int t = r - 1; t >= 0; --t) {
        if (n <= kLeaf) {
          exists = false;
          break;
        }
        const int64_t h = pw_split(n);
        if ((q >> t) & 1) {
          lo += h;
          n -= h;
        } else {
          n = h;
        }
      }
      const int vi = cnt - 1 + q;
      kind[vi] = !exists ? 0 : (n <= kLeaf ? 1 : 2);
      if (exists && n <= kLeaf) {
        const int k = atomicAdd(&nleaf, 1);
        leaf_lo[k] = (int)lo;
        leaf_n[k] = (int)n;
        leaf_v[k] = vi;
      }
    }
  }
  __syncthreads();
  // B: leaves, 8 lanes each (lane k owns numpy's accumulator r[k]: conflict-free
  // shared-memory rows), combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by shuffles
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane & 7;
    const int nw = blockDim.x >> 5;
    for (int L0 = warp * 4; L0 < nleaf; L0 += nw * 4) {
      const int L = L0 + (lane >> 3);
      const bool act = L < nleaf;
      const int lo = act ? leaf_lo[L] : 0, n = act ? leaf_n[L] : 0;
      double r = 0.0;
      const int body = n >= 8 ? n - (n % 8) : 0;
      if (body > 0) {
        r = a[lo + sub];
        for (int i = 8; i < body; i += 8) r = __dadd_rn(r, a[lo + i + sub]);
      }
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
      if (act && sub == 0) {
        double res = body > 0 ? r : 0.0;
        for (int i = body; i < n; ++i) res = __dadd_rn(res, a[lo + i]);
        V[leaf_v[L]] = res;
      }
    }
  }
  __syncthreads();
  // C: internal nodes bottom-up
  for (int r = rdepth - 1; r >= 0; --r) {
    const int cnt = 1 << r;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
      const int vi = cnt - 1 + q;
      if (kind[vi] == 2) {
        const int ci = 2 * cnt - 1 + 2 * q;
        V[vi] = __dadd_rn(V[ci], V[ci + 1]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) vals[b * ((int64_t)1 << t1) + node] = V[0];
}

// ------------------------------------------------- pairwise total: tiers
// Every node above depth t1 is internal, so the tree between t_out and t_in
// is complete: parent = left + right, folded level by level.
__global__ void __launch_bounds__(256) k_pp_tier(const double* __restrict__ in, int t_in,
                                                  double* __restrict__ out, int t_out,
                                                  const int32_t* __restrict__ halted, int64_t j) {
  __shared__ double A[1 << kTierLevels];
  __shared__ double Bf[1 << (kTierLevels - 1)];
  const int b = blockIdx.y;
  if (halted && halted[b] < j) return;
  const int L = t_in - t_out;
  const int cnt = 1 << L;
  const double* src = in + b * ((int64_t)1 << t_in) + (int64_t)blockIdx.x * cnt;
  for (int q = threadIdx.x; q < cnt; q += blockDim.x) A[q] = src[q];
  __syncthreads();
  double* s = A;
  double* dst = Bf;
  for (int l = L; l > 0; --l) {
    const int half = 1 << (l - 1);
    for (int q = threadIdx.x; q < half; q += blockDim.x) dst[q] = __dadd_rn(s[2 * q], s[2 * q + 1]);
    __syncthreads();
    double* tmp = s;
    s = dst;
    dst = tmp;
  }
  if (threadIdx.x == 0) out[b * ((int64_t)1 << t_out) + blockIdx.x] = s[0];
}

// Rigorous bound on |cdf_i - r_i| (see the file header / DESIGN.md):
// numpy's cdf_i = fl(S_i / S_last), S the serial cumsum of p_j = fl(m_j/total);
// r_i = A_i / A_N the exact prefix ratio of min_d2.
FK_DEV double pp_margin(double i, double N, double r) {
  if (!(r > 0.0)) return 0.0;  // A_i == 0: every p_j (j<=i) is 0, so cdf_i == 0 exactly
  const double u = 0x1p-53;
  const double core = (1.0 - r + 4.0 * u) * i * r + r * (N - i);
  const double D = u * (1.0 + 8.0 * N * u) * core + 8.0 * u * r + 0x1p-90 * r;
  return D * (1.0 + 0x1p-30) + 1e-300;
}

// ---------------------------------------------------------------- select
// One CTA (1024 threads) per batch element.  Finds i* = first i with
// A_i > u * A_N and certifies that numpy's searchsorted(cdf, u, "right") is
// i*; otherwise raises flag[b] for k_pp_exact.
__global__ void __launch_bounds__(1024) k_pp_select(
    const double* __restrict__ m, int64_t N, int64_t m_sb, int t1,
    const double* __restrict__ root, const double2* __restrict__ ddsum,
    const double* __restrict__ u, int64_t K, int64_t j, int64_t* __restrict__ idx,
    int32_t* __restrict__ halted, int32_t* __restrict__ flag, double* __restrict__ totals,
    int force_exact) {
  __shared__ DD wb[32];
  __shared__ int64_t s_blk;
  __shared__ DD s_pre;
  __shared__ int s_first;
  __shared__ DD s_ai, s_aim1;
  const int b = blockIdx.x;
  if (halted[b] < j) return;
  const double total = root[b];
  if (!(total > 0.0)) {  // reference: rng.integers(n) from here on (host side)
    if (threadIdx.x == 0) {
      halted[b] = (int32_t)j;
      flag[b] = 0;
    }
    return;
  }
  const double ud = u[b * (K - 1) + (j - 1)];
  const int64_t nb = (int64_t)1 << t1;
  const int64_t g = (nb + blockDim.x - 1) / blockDim.x;
  const int64_t k0 = i64min(nb, (int64_t)threadIdx.x * g), k1 = i64min(nb, k0 + g);
  const double2* ds = ddsum + b * nb;
  DD mine{0.0, 0.0};
  for (int64_t k = k0; k < k1; ++k) mine = dd_add(mine, DD{ds[k].x, ds[k].y});
  if (threadIdx.x == 0) {
    s_blk = INT64_MAX;
    s_first = INT32_MAX;
  }
  DD AN;
  const DD excl = block_excl_scan(mine, wb, &AN);
  const DD Y = dd_mul1(AN, ud);
  const DD incl = dd_add(excl, mine);
  int64_t my_blk = -1;
  DD my_pre{0.0, 0.0};
  if (k0 < k1 && dd_le(excl, Y) && dd_gt(incl, Y)) {
    DD pre = excl;
    for (int64_t k = k0; k < k1; ++k) {
      const DD nx = dd_add(pre, DD{ds[k].x, ds[k].y});
      if (dd_gt(nx, Y)) {
        my_blk = k;
        my_pre = pre;
        atomicMin(reinterpret_cast<unsigned long long*>(&s_blk), (unsigned long long)k);
        break;
      }
      pre = nx;
    }
  }
  __syncthreads();
  if (my_blk >= 0 && my_blk == s_blk) s_pre = my_pre;
  __syncthreads();
  const int64_t blk = s_blk;
  bool ok = blk != INT64_MAX;
  int64_t lo = 0, n = 0;
  if (ok) {
    pw_walk(N, t1, blk, lo, n);
    const double* src = m + b * m_sb + lo;
    const int per = (int)((n + blockDim.x - 1) / blockDim.x);  // <= 4
    const int e0 = threadIdx.x * per;
    double v[4];
    DD loc{0.0, 0.0};
    for (int q = 0; q < per; ++q) {
      v[q] = (e0 + q < n) ? src[e0 + q] : 0.0;
      loc = dd_add1(loc, v[q]);
    }
    DD tot;
    const DD base0 = block_excl_scan(loc, wb, &tot);
    const DD base = dd_add(s_pre, base0);
    DD run = base;
    for (int q = 0; q < per; ++q) {
      if (e0 + q >= n) break;
      const DD nx = dd_add1(run, v[q]);
      if (dd_gt(nx, Y)) {
        atomicMin(&s_first, e0 + q);
        break;
      }
      run = nx;
    }
    __syncthreads();
    ok = s_first != INT32_MAX;
    if (ok) {
      const int f = s_first;
      if (f >= e0 && f < e0 + per) {  // the unique owner of element f
        DD r2 = base;
        for (int q = 0; q < f - e0; ++q) r2 = dd_add1(r2, v[q]);
        s_aim1 = r2;
        s_ai = dd_add1(r2, v[f - e0]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bool cert = ok && !force_exact;
    if (cert) {
      const int64_t is = lo + s_first;
      const double an = AN.hi + AN.lo;
      const double rh = (s_ai.hi + s_ai.lo) / an;
      const double rl = (s_aim1.hi + s_aim1.lo) / an;
      const double Nd = (double)N;
      cert = (rh - pp_margin((double)is, Nd, rh) > ud) &&
             (is == 0 || rl + pp_margin((double)(is - 1), Nd, rl) <= ud);
      if (cert) idx[b * K + j] = is;
    }
    flag[b] = cert ? 0 : 1;
    totals[b] = total;
  }
}

// ------------------------------------------------- exact serial fallback
// Literal numpy: p = m / total; cdf = cumsum(p); cdf /= cdf[-1];
// searchsorted(cdf, u, side="right").  Warps 1.. compute the next tile of p
// while lane 0 of warp 0 runs the serial chain over the current one.
__global__ void __launch_bounds__(256) k_pp_exact(const double* __restrict__ m, int64_t N,
                                                   int64_t m_sb, const double* __restrict__ u,
                                                   int64_t K, int64_t j, int64_t* __restrict__ idx,
                                                   const int32_t* __restrict__ halted,
                                                   const int32_t* __restrict__ flag,
                                                   const double* __restrict__ totals,
                                                   double* __restrict__ ckpt, int64_t ck_sb) {
  __shared__ double buf[2][kExactTile];
  __shared__ double s_last;
  __shared__ int64_t s_tile;
  const int b = blockIdx.x;
  if (halted[b] <= j || !flag[b]) return;
  const double total = totals[b];
  const double ud = u[b * (K - 1) + (j - 1)];
  const double* src = m + b * m_sb;
  double* ck = ckpt + b * ck_sb;
  const int64_t ntiles = (N + kExactTile - 1) / kExactTile;
  for (int64_t k = threadIdx.x; k < i64min(N, kExactTile); k += blockDim.x)
    buf[0][k] = __ddiv_rn(src[k], total);
  __syncthreads();
  double S = 0.0;
  for (int64_t t = 0; t < ntiles; ++t) {
    const int64_t base = t * kExactTile;
    const int len = (int)i64min(kExactTile, N - base);
    if (threadIdx.x >= 32) {
      if (t + 1 < ntiles) {
        const int64_t nb = base + kExactTile;
        const int nl = (int)i64min(kExactTile, N - nb);
        double* dst = buf[(t + 1) & 1];
        for (int k = threadIdx.x - 32; k < nl; k += blockDim.x - 32)
          dst[k] = __ddiv_rn(src[nb + k], total);
      }
    } else if (threadIdx.x == 0) {
      const double* p = buf[t & 1];
      int k = 0;
      for (; k + 8 <= len; k += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = p[k + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) S = __dadd_rn(S, v[q]);
      }
      for (; k < len; ++k) S = __dadd_rn(S, p[k]);
      ck[t] = S;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    s_last = S;
    s_tile = ntiles - 1;
  }
  __syncthreads();
  const double Sl = s_last;
  for (int64_t t = threadIdx.x; t < ntiles; t += blockDim.x)
    if (__ddiv_rn(ck[t], Sl) > ud) atomicMin(reinterpret_cast<unsigned long long*>(&s_tile),
                                             (unsigned long long)t);
  __syncthreads();
  const int64_t t = s_tile;
  const int64_t base = t * kExactTile;
  const int len = (int)i64min(kExactTile, N - base);
  for (int k = threadIdx.x; k < len; k += blockDim.x) buf[0][k] = __ddiv_rn(src[base + k], total);
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = t > 0 ? ck[t - 1] : 0.0;
    int64_t ans = base + len - 1;
    for (int k = 0; k < len; ++k) {
      s = __dadd_rn(s, buf[0][k]);
      if (__ddiv_rn(s, Sl) > ud) {
        ans = base + k;
        break;
      }
    }
    idx[b * K + j] = ans;
  }
}

// ----------------------------------------- exact cumsum in parallel (fallback)
// numpy's cdf = cumsum(p) is the serial chain S_k = fl(S_{k-1} + p_k).  While
// S stays in one binade [2^e, 2^(e+1)) it is a multiple of q = 2^(e-52) and
// fl(S + p) = S + q*inc, inc = p/q rounded to nearest with ties to an even
// S'/q -- a function of the parity of S/q only.  A run of elements is thus a
// composable function F(parity) = (increment, end parity).  k_ex_tiles forms
// p = fl(m/total) and exact per-tile sums; its last block scans them to
// predict each tile's starting binade.  k_ex_funcs builds every tile's F for
// its predicted binade in parallel; its last block walks the tiles applying F
// where the prediction holds and no binade crossing happens inside the tile
// (s + inc < 2^53, S monotone), and replays the few other tiles literally.
// Every step reproduces fl(S + p) exactly, so the walk equals numpy's chain.
struct RFun {
  long long inc0, inc1;
  int out0, out1, big;
};
FK_DEV long long sat_add(long long a, long long b) {
  const long long c = a + b;
  return c > (1LL << 62) ? (1LL << 62) : c;
}
FK_DEV RFun rf_identity() { return {0, 0, 0, 1, 0}; }
FK_DEV RFun rf_compose(const RFun& f, const RFun& g) {  // f, then g
  RFun h;
  h.inc0 = sat_add(f.inc0, f.out0 ? g.inc1 : g.inc0);
  h.out0 = f.out0 ? g.out1 : g.out0;
  h.inc1 = sat_add(f.inc1, f.out1 ? g.inc1 : g.inc0);
  h.out1 = f.out1 ? g.out1 : g.out0;
  h.big = f.big | g.big;
  return h;
}
FK_DEV RFun rf_element(double p, int e) {
  const double r = scalbn(p, 52 - e);  // p / q, exact
  RFun f;
  f.big = 0;
  if (!(r < 9007199254740992.0)) {  // >= 2^53 (or inf): crosses by itself
    f.inc0 = f.inc1 = 1LL << 62;
    f.out0 = f.out1 = 0;
    f.big = 1;
    return f;
  }
  const double A = floor(r);
  const double fr = r - A;
  const long long a = (long long)A;
  if (fr == 0.5) {  // tie: the even neighbour of s + a + 1/2
    f.inc0 = a + (a & 1);
    f.inc1 = a + ((a + 1) & 1);
    f.out0 = f.out1 = 0;
    return f;
  }
  f.inc0 = f.inc1 = fr > 0.5 ? a + 1 : a;
  f.out0 = (int)(f.inc0 & 1);
  f.out1 = (int)((f.inc1 + 1) & 1);
  return f;
}
FK_DEV RFun rf_shfl_down(const RFun& f, int off) {
  RFun g;
  g.inc0 = __shfl_down_sync(0xffffffffu, f.inc0, off);
  g.inc1 = __shfl_down_sync(0xffffffffu, f.inc1, off);
  g.out0 = __shfl_down_sync(0xffffffffu, f.out0, off);
  g.out1 = __shfl_down_sync(0xffffffffu, f.out1, off);
  g.big = __shfl_down_sync(0xffffffffu, f.big, off);
  return g;
}

constexpr int kExThreads = 256;
constexpr int kExPer = kExactTile / kExThreads;  // 8 elements per thread
constexpr int kNoBinade = -100000;

// Last block of a grid to arrive (after a __threadfence) returns true.
FK_DEV bool last_block_done(unsigned int* counter, unsigned int nblocks) {
  __shared__ unsigned int s_ticket;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_ticket = atomicAdd(counter, 1u);
  __syncthreads();
  const bool last = s_ticket == nblocks - 1;
  if (last && threadIdx.x == 0) *counter = 0;  // reset for the next draw
  __threadfence();
  return last;
}

__global__ void __launch_bounds__(kExThreads) k_ex_tiles(
    const double* __restrict__ m, int64_t N, const int32_t* __restrict__ halted,
    const int32_t* __restrict__ flag, const double* __restrict__ totals, int64_t j,
    double* __restrict__ p, double2* __restrict__ tsum, int* __restrict__ epred,
    unsigned int* __restrict__ counter) {
  __shared__ DD wb[32];
  const int b = blockIdx.y;
  if (halted[b] <= j || !flag[b]) return;
  const int64_t ntiles = gridDim.x, t = blockIdx.x;
  const double total = totals[b];
  const int64_t k0 = t * kExactTile + threadIdx.x * kExPer;
  DD acc{0.0, 0.0};
#pragma unroll
  for (int q = 0; q < kExPer; ++q) {
    const int64_t k = k0 + q;
    if (k < N) {
      const double v = __ddiv_rn(m[(int64_t)b * N + k], total);
      p[(int64_t)b * N + k] = v;
      acc = dd_add1(acc, v);
    }
  }
  DD tot;
  (void)block_excl_scan(acc, wb, &tot);
  if (threadIdx.x == 0) tsum[(int64_t)b * ntiles + t] = make_double2(tot.hi, tot.lo);
  if (!last_block_done(counter + 2 * b, (unsigned)ntiles)) return;
  // exclusive prefix of the tile sums -> predicted binade at each tile start
  const double2* ts = tsum + (int64_t)b * ntiles;
  DD carry{0.0, 0.0};
  for (int64_t base = 0; base < ntiles; base += kExThreads) {
    const int64_t tt = base + threadIdx.x;
    const DD v = tt < ntiles ? DD{ts[tt].x, ts[tt].y} : DD{0.0, 0.0};
    DD chunk;
    const DD ex = dd_add(carry, block_excl_scan(v, wb, &chunk));
    if (tt < ntiles) {
      const double sp = ex.hi + ex.lo;
      epred[(int64_t)b * ntiles + tt] = sp >= 0x1p-1000 ? ilogb(sp) : kNoBinade;
    }
    carry = dd_add(carry, chunk);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kExThreads) k_ex_funcs(
    const double* __restrict__ p, int64_t N, const double* __restrict__ u, int64_t K, int64_t j,
    int64_t* __restrict__ idx, const int32_t* __restrict__ halted,
    const int32_t* __restrict__ flag, const int* __restrict__ epred, RFun* __restrict__ F,
    double* __restrict__ ckpt, unsigned int* __restrict__ counter) {
  __shared__ RFun wf[kExThreads / 32];
  __shared__ double tp[kExactTile];
  __shared__ RFun sF[kExThreads];
  __shared__ int sE[kExThreads];
  __shared__ int64_t s_slow, s_pos;
  __shared__ double s_S;
  const int b = blockIdx.y;
  if (halted[b] <= j || !flag[b]) return;
  const int64_t ntiles = gridDim.x, t = blockIdx.x;
  const double* pb = p + (int64_t)b * N;
  const int e = epred[(int64_t)b * ntiles + t];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  RFun f = rf_identity();
  if (e != kNoBinade) {
    const int64_t k0 = t * kExactTile + threadIdx.x * kExPer;
#pragma unroll
    for (int q = 0; q < kExPer; ++q)
      if (k0 + q < N) f = rf_compose(f, rf_element(pb[k0 + q], e));
  } else {
    f.big = 1;
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {  // ordered: lane i's run precedes lane i+off's
    const RFun g = rf_shfl_down(f, off);
    if ((lane & (2 * off - 1)) == 0) f = rf_compose(f, g);
  }
  if (lane == 0) wf[warp] = f;
  __syncthreads();
  if (threadIdx.x == 0) {
    RFun h = wf[0];
    for (int w = 1; w < kExThreads / 32; ++w) h = rf_compose(h, wf[w]);
    F[(int64_t)b * ntiles + t] = h;
  }
  if (!last_block_done(counter + 2 * b, (unsigned)ntiles)) return;
  // ---- the walk (one block): fast tiles apply F, the others are replayed
  const RFun* Fb = F + (int64_t)b * ntiles;
  const int* Eb = epred + (int64_t)b * ntiles;
  double* ck = ckpt + (int64_t)b * ntiles;
  if (threadIdx.x == 0) s_S = 0.0;
  for (int64_t c0 = 0; c0 < ntiles; c0 += kExThreads) {
    const int64_t cn = i64min(kExThreads, ntiles - c0);
    if (threadIdx.x < cn) {
      sF[threadIdx.x] = Fb[c0 + threadIdx.x];
      sE[threadIdx.x] = Eb[c0 + threadIdx.x];
    }
    if (threadIdx.x == 0) s_pos = 0;
    __syncthreads();
    while (s_pos < cn) {
      if (threadIdx.x == 0) {
        double S = s_S;
        int64_t i = s_pos;
        s_slow = -1;
        for (; i < cn; ++i) {
          const RFun& h = sF[i];
          bool fast = false;
          if (!h.big && S >= 0x1p-1000 && ilogb(S) == sE[i]) {
            const int ee = sE[i];
            const long long sv = (long long)scalbn(S, 52 - ee);
            const int par = (int)(sv & 1);
            const long long s2 = sat_add(sv, par ? h.inc1 : h.inc0);
            if (s2 < (1LL << 53)) {
              S = scalbn((double)s2, ee - 52);
              fast = true;
            }
          }
          if (!fast) {
            s_slow = c0 + i;
            break;
          }
          ck[c0 + i] = S;
        }
        s_S = S;
        s_pos = i;
      }
      __syncthreads();
      const int64_t slow = s_slow;
      if (slow >= 0) {  // replay this tile literally: S = fl(S + p_k)
        const int64_t base = slow * kExactTile;
        const int len = (int)i64min(kExactTile, N - base);
        for (int k = threadIdx.x; k < len; k += kExThreads) tp[k] = pb[base + k];
        __syncthreads();
        if (threadIdx.x == 0) {
          double S = s_S;
          for (int k = 0; k < len; ++k) S = __dadd_rn(S, tp[k]);
          s_S = S;
          ck[slow] = S;
          s_pos = s_pos + 1;
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
  // ---- searchsorted(cumsum / cumsum[-1], u, "right"): first tile, then element
  __shared__ int64_t s_tile;
  const double Sl = s_S;
  const double ud = u[b * (K - 1) + (j - 1)];
  if (threadIdx.x == 0) s_tile = ntiles - 1;
  __syncthreads();
  for (int64_t tt = threadIdx.x; tt < ntiles; tt += kExThreads)
    if (__ddiv_rn(ck[tt], Sl) > ud)
      atomicMin(reinterpret_cast<unsigned long long*>(&s_tile), (unsigned long long)tt);
  __syncthreads();
  const int64_t tt = s_tile;
  const int64_t base = tt * kExactTile;
  const int len = (int)i64min(kExactTile, N - base);
  for (int k = threadIdx.x; k < len; k += kExThreads) tp[k] = pb[base + k];
  __syncthreads();
  if (threadIdx.x == 0) {
    double S = tt > 0 ? ck[tt - 1] : 0.0;
    int64_t ans = base + len - 1;
    for (int k = 0; k < len; ++k) {
      S = __dadd_rn(S, tp[k]);
      if (__ddiv_rn(S, Sl) > ud) {
        ans = base + k;
        break;
      }
    }
    idx[b * K + j] = ans;
  }
}

__global__ void k_pp_init(int32_t* halted, int32_t* flag, unsigned int* counters, int64_t B,
                          int64_t K) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) {
    halted[b] = (int32_t)K;
    flag[b] = 0;
    counters[2 * b] = 0;
    counters[2 * b + 1] = 0;
  }
}

// ------------------------------------------------------------------- plan
struct Plan {
  int t1 = 0;      // depth of the bottom nodes
  int rdepth = 0;  // deepest leaf below t1 (relative)
  bool valid = true;
  std::vector<int> tiers;  // t_in sequence: t1 -> ... -> 0
};

Plan make_plan(int64_t N) {
  Plan p;
  // distinct node sizes per depth (the set stays tiny)
  std::vector<int64_t> level{N};
  int depth = 0, t1 = -1, maxdepth = 0;
  while (true) {
    int64_t mx = 0, mn = INT64_MAX;
    bool any_internal = false;
    for (int64_t s : level) {
      mx = std::max(mx, s);
      mn = std::min(mn, s);
      if (s > kLeaf) any_internal = true;
    }
    if (t1 < 0 && mx <= kNodeMax) t1 = depth;
    if (t1 < 0 && mn <= kLeaf) p.valid = false;  // a leaf above t1: tiers would be incomplete
    if (!any_internal) {
      maxdepth = depth;
      break;
    }
    std::vector<int64_t> nxt;
    for (int64_t s : level) {
      if (s <= kLeaf) continue;
      const int64_t h = pw_split(s);
      nxt.push_back(h);
      nxt.push_back(s - h);
    }
    std::sort(nxt.begin(), nxt.end());
    nxt.erase(std::unique(nxt.begin(), nxt.end()), nxt.end());
    level.swap(nxt);
    ++depth;
  }
  p.t1 = t1;
  p.rdepth = maxdepth - t1;
  int t = t1;
  while (t > 0) {
    p.tiers.push_back(t);
    t = std::max(0, t - kTierLevels);
  }
  return p;
}

bool exact_serial_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FK_PP_EXACT_SERIAL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

bool force_exact_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FK_PP_FORCE_EXACT");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

struct WsLayout {
  size_t vals, vals2, root, dd, totals, flag, ckpt, p, tsum, epred, fun, counters, bytes;
  int64_t ntiles;
};

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

WsLayout ws_layout(int64_t B, int64_t N) {
  const Plan p = make_plan(N);
  WsLayout w;
  const size_t nb = (size_t)1 << p.t1;
  w.ntiles = (N + kExactTile - 1) / kExactTile;
  size_t o = 0;
  w.vals = o; o += al256(B * nb * 8);
  w.vals2 = o; o += al256(B * std::max<size_t>(1, nb >> kTierLevels) * 8 + 8 * B);
  w.root = o; o += al256(B * 8);
  w.dd = o; o += al256(B * nb * 16);
  w.totals = o; o += al256(B * 8);
  w.flag = o; o += al256(B * 4);
  w.ckpt = o; o += al256(B * w.ntiles * 8);
  w.p = o; o += al256((size_t)B * N * 8);           // fallback: p = fl(m / total)
  w.tsum = o; o += al256(B * w.ntiles * 16);
  w.epred = o; o += al256(B * w.ntiles * 4);
  w.fun = o; o += al256(B * w.ntiles * sizeof(RFun));
  w.counters = o; o += al256(B * 2 * 4);
  w.bytes = o;
  return w;
}

int sweep_variant() {  // FK_PP_SWEEP=pipe selects the persistent cp.async ring (A/B runs)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FK_PP_SWEEP");
    v = (e && e[0] == 'p') ? 1 : 0;
  }
  return v;
}

template <typename T, int D>
cudaError_t sweep_fast(const T* Xt, int64_t B, int64_t rows, int d, int64_t x_sb, const T* Ct,
                       int64_t cen_sb, const int64_t* idx, int64_t K, int64_t col, double* m,
                       int64_t m_sb, int first, const int32_t* halted, int64_t j, cudaStream_t s,
                       size_t cbytes, int stride_b) {
  const size_t tile_b = (size_t)kSweepRows * stride_b;
  const int se = stride_b / (int)sizeof(T);
  if (sweep_variant() == 1 && cbytes + 2 * tile_b <= 220 * 1024) {
    const int stages = cbytes + 3 * tile_b <= 110 * 1024 ? 3 : 2;
    const size_t sm = cbytes + stages * tile_b;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = stages == 3 ? 2 : 1;
    const int64_t ntiles = (rows + kSweepRows - 1) / kSweepRows;
    const int64_t gx = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sms * per_sm / B));
    dim3 grid((unsigned)gx, (unsigned)B);
    if (stages == 3) {
      cudaFuncSetAttribute(k_pp_sweep_pipe<T, 3, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_pp_sweep_pipe<T, 3, D><<<grid, kSweepRows, sm, s>>>(Xt, rows, d, x_sb, Ct, cen_sb, idx, K, col,
                                                           m, m_sb, first, halted, j, se);
    } else {
      cudaFuncSetAttribute(k_pp_sweep_pipe<T, 2, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_pp_sweep_pipe<T, 2, D><<<grid, kSweepRows, sm, s>>>(Xt, rows, d, x_sb, Ct, cen_sb, idx, K, col,
                                                           m, m_sb, first, halted, j, se);
    }
    return cudaGetLastError();
  }
  const size_t smem = cbytes + tile_b;
  cudaFuncSetAttribute(k_pp_sweep<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  dim3 grid((unsigned)((rows + kSweepRows - 1) / kSweepRows), (unsigned)B);
  k_pp_sweep<T, D><<<grid, kSweepRows, smem, s>>>(Xt, rows, d, x_sb, Ct, cen_sb, idx, K, col, m, m_sb,
                                                  first, halted, j, se);
  return cudaGetLastError();
}

template <typename T>
cudaError_t sweep_t(const void* X, int64_t B, int64_t rows, int d, int64_t x_sb, const void* cen,
                    int64_t cen_sb, const int64_t* idx, int64_t K, int64_t col, double* m,
                    int64_t m_sb, int first, const int32_t* halted, int64_t j, cudaStream_t s) {
  const size_t cbytes = ((size_t)d * 8 + 15) & ~size_t(15);
  const int rb = d * (int)sizeof(T);
  const int stride_b = ((rb + 15) & ~15) + 16;  // padded: conflict-free 16-B row reads
  const size_t smem = cbytes + (size_t)kSweepRows * stride_b;
  const T* Xt = static_cast<const T*>(X);
  const T* Ct = static_cast<const T*>(cen);
  if (rows <= 0) return cudaSuccess;
  const bool vec = (rb & 15) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                   ((x_sb * (int64_t)sizeof(T)) & 15) == 0;
  if (vec && smem <= 200 * 1024) {
#define FK_PP_FAST(DV)                                                                          \
  return sweep_fast<T, DV>(Xt, B, rows, d, x_sb, Ct, cen_sb, idx, K, col, m, m_sb, first, halted, \
                           j, s, cbytes, stride_b)
    switch (d) {
      case 16: FK_PP_FAST(16);
      case 32: FK_PP_FAST(32);
      case 64: FK_PP_FAST(64);
      case 128: FK_PP_FAST(128);
      case 192: FK_PP_FAST(192);
      case 256: FK_PP_FAST(256);
      default: FK_PP_FAST(0);
    }
#undef FK_PP_FAST
  }
  if (smem <= 200 * 1024) {
    cudaFuncSetAttribute(k_pp_sweep<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    dim3 grid((unsigned)((rows + kSweepRows - 1) / kSweepRows), (unsigned)B);
    k_pp_sweep<T, 0><<<grid, kSweepRows, smem, s>>>(Xt, rows, d, x_sb, Ct, cen_sb, idx, K, col, m,
                                                    m_sb, first, halted, j, stride_b / (int)sizeof(T));
  } else if (vec && cbytes <= 200 * 1024) {
    cudaFuncSetAttribute(k_pp_sweep_global<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    dim3 grid((unsigned)((rows + 127) / 128), (unsigned)B);
    k_pp_sweep_global<T><<<grid, 128, cbytes, s>>>(Xt, rows, d, x_sb, Ct, cen_sb, idx, K, col, m,
                                                   m_sb, first, halted, j);
  } else {
    if (cbytes > 200 * 1024) return cudaErrorInvalidValue;
    cudaFuncSetAttribute(k_pp_sweep_scalar<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    dim3 grid((unsigned)((rows + 127) / 128), (unsigned)B);
    k_pp_sweep_scalar<T><<<grid, 128, cbytes, s>>>(Xt, rows, d, x_sb, Ct, cen_sb, idx, K, col, m,
                                                   m_sb, first, halted, j);
  }
  return cudaGetLastError();
}

cudaError_t sweep_dispatch(int dt, const void* X, int64_t B, int64_t rows, int d, int64_t x_sb,
                           const void* cen, int64_t cen_sb, const int64_t* idx, int64_t K,
                           int64_t col, double* m, int64_t m_sb, int first, const int32_t* halted,
                           int64_t j, cudaStream_t s) {
  switch (dt) {
    case DT_F32:
      return sweep_t<float>(X, B, rows, d, x_sb, cen, cen_sb, idx, K, col, m, m_sb, first, halted, j, s);
    case DT_F64:
      return sweep_t<double>(X, B, rows, d, x_sb, cen, cen_sb, idx, K, col, m, m_sb, first, halted, j, s);
    case DT_BF16:
      return sweep_t<__nv_bfloat16>(X, B, rows, d, x_sb, cen, cen_sb, idx, K, col, m, m_sb, first,
                                    halted, j, s);
    case DT_F16:
      return sweep_t<__half>(X, B, rows, d, x_sb, cen, cen_sb, idx, K, col, m, m_sb, first, halted,
                             j, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// In-core pruning state behind the base layout: nearest-center ids (B,N),
// chosen centers in f64 (B,K,d) and center-to-center distances (B,K).
size_t pruning_bytes(int64_t B, int64_t N, int64_t K, int64_t d) {
  if (K <= 0 || d <= 0) return 0;
  return al256((size_t)B * N * 4) + al256((size_t)B * K * d * 8) + al256((size_t)B * K * 8);
}

size_t kmeanspp_workspace_bytes(int64_t B, int64_t N, int64_t K, int64_t d) {
  return ws_layout(B, N).bytes + pruning_bytes(B, N, K, d);
}

// Opt-in (FK_PP_PRUNE=1): on the config-3 blob data the pruned sweep is
// slower (0.62 vs 0.55 ms per draw at N=8M, K=1024: in 128 dimensions the
// triangle bound rarely clears rows of clusters without a center yet), so the
// plain sweep is the default; data that prunes well can turn it on.
bool prune_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FK_PP_PRUNE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

template <typename T, int D>
cudaError_t sweep_pruned_t(const void* X, int64_t B, int64_t N, int d, const int64_t* idx,
                           int64_t K, int64_t col, double* m, int32_t* nearest,
                           const double* cdist, int first, const int32_t* halted, int64_t j,
                           cudaStream_t s) {
  const size_t cbytes = ((size_t)d * 8 + 15) & ~size_t(15);
  const int rb = d * (int)sizeof(T);
  const int stride_b = ((rb + 15) & ~15) + 16;
  const size_t smem = cbytes + (size_t)kSweepRows * stride_b;
  cudaFuncSetAttribute(k_pp_sweep_pruned<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       200 * 1024);
  dim3 grid((unsigned)((N + kSweepRows - 1) / kSweepRows), (unsigned)B);
  k_pp_sweep_pruned<T, D><<<grid, kSweepRows, smem, s>>>(static_cast<const T*>(X), N, d, idx, K, col,
                                                         m, nearest, cdist, first, halted, j,
                                                         stride_b / (int)sizeof(T));
  return cudaGetLastError();
}

template <typename T>
cudaError_t sweep_pruned_d(const void* X, int64_t B, int64_t N, int d, const int64_t* idx,
                           int64_t K, int64_t col, double* m, int32_t* nearest,
                           const double* cdist, int first, const int32_t* halted, int64_t j,
                           cudaStream_t s) {
#define FK_PP_PR(DV) \
  return sweep_pruned_t<T, DV>(X, B, N, d, idx, K, col, m, nearest, cdist, first, halted, j, s)
  switch (d) {
    case 16: FK_PP_PR(16);
    case 32: FK_PP_PR(32);
    case 64: FK_PP_PR(64);
    case 128: FK_PP_PR(128);
    case 192: FK_PP_PR(192);
    case 256: FK_PP_PR(256);
    default: FK_PP_PR(0);
  }
#undef FK_PP_PR
}

cudaError_t sweep_pruned(int dt, const void* X, int64_t B, int64_t N, int d, const int64_t* idx,
                         int64_t K, int64_t col, double* m, int32_t* nearest, const double* cdist,
                         int first, const int32_t* halted, int64_t j, cudaStream_t s) {
  switch (dt) {
    case DT_F32: return sweep_pruned_d<float>(X, B, N, d, idx, K, col, m, nearest, cdist, first, halted, j, s);
    case DT_F64: return sweep_pruned_d<double>(X, B, N, d, idx, K, col, m, nearest, cdist, first, halted, j, s);
    case DT_BF16:
      return sweep_pruned_d<__nv_bfloat16>(X, B, N, d, idx, K, col, m, nearest, cdist, first, halted, j, s);
    case DT_F16: return sweep_pruned_d<__half>(X, B, N, d, idx, K, col, m, nearest, cdist, first, halted, j, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_kmeanspp_init(int32_t* halted, void* ws, int64_t B, int64_t N, int64_t K,
                                 cudaStream_t s) {
  const WsLayout w = ws_layout(B, N);
  int32_t* flag = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + w.flag);
  unsigned int* counters = reinterpret_cast<unsigned int*>(static_cast<uint8_t*>(ws) + w.counters);
  k_pp_init<<<(unsigned)((B + 255) / 256), 256, 0, s>>>(halted, flag, counters, B, K);
  return cudaGetLastError();
}

cudaError_t launch_kmeanspp_sweep(int dt, const void* X, int64_t B, int64_t rows, int64_t d,
                                  int64_t x_sb, const void* cen, int64_t cen_sb,
                                  const int64_t* idx, int64_t K, int64_t col, double* m,
                                  int64_t m_sb, int first, const int32_t* halted, int64_t j,
                                  cudaStream_t s) {
  return sweep_dispatch(dt, X, B, rows, (int)d, x_sb, cen, cen_sb, idx, K, col, m, m_sb, first,
                        halted, j, s);
}

// numpy's pairwise sum (np.sum of a contiguous float64 array) of every row of
// the (B, N) table m -- the objective of f64 data (pipeline._objective_row):
// the bottom nodes and tiers of the k-means++ total, no selection.  Returns
// cudaErrorInvalidValue for the (tiny) sizes the node plan does not cover.
size_t pairwise_total_workspace(int64_t B, int64_t N) {
  const Plan p = make_plan(N);
  const size_t nb = (size_t)1 << p.t1;
  return al256(B * nb * 8) + al256(B * std::max<size_t>(1, nb >> kTierLevels) * 8 + 8 * B) +
         al256(B * nb * 16);
}

cudaError_t launch_pairwise_total(const double* m, int64_t B, int64_t N, double* out, void* ws,
                                  cudaStream_t s) {
  const Plan p = make_plan(N);
  if (!p.valid || p.rdepth > kNodeLevels) return cudaErrorInvalidValue;
  const size_t nb = (size_t)1 << p.t1;
  uint8_t* base = static_cast<uint8_t*>(ws);
  double* vals = reinterpret_cast<double*>(base);
  double* vals2 = reinterpret_cast<double*>(base + al256(B * nb * 8));
  double2* dd = reinterpret_cast<double2*>(base + al256(B * nb * 8) +
                                           al256(B * std::max<size_t>(1, nb >> kTierLevels) * 8 + 8 * B));
  dim3 g1((unsigned)nb, (unsigned)B);
  k_pp_node<<<g1, 256, 0, s>>>(m, N, N, p.t1, p.rdepth, nullptr, 0, p.t1 == 0 ? out : vals, dd);
  const double* in = vals;
  for (size_t k = 0; k < p.tiers.size(); ++k) {
    const int t_in = p.tiers[k];
    const int t_out = std::max(0, t_in - kTierLevels);
    double* o = t_out == 0 ? out : ((k & 1) ? vals : vals2);
    dim3 g((unsigned)((int64_t)1 << t_out), (unsigned)B);
    k_pp_tier<<<g, 256, 0, s>>>(in, t_in, o, t_out, nullptr, 0);
    in = o;
  }
  return cudaGetLastError();
}

cudaError_t launch_kmeanspp_select(const double* m, int64_t B, int64_t N, const double* u,
                                   int64_t K, int64_t j, int64_t* idx, int32_t* halted, void* ws,
                                   cudaStream_t s) {
  const Plan p = make_plan(N);
  const WsLayout w = ws_layout(B, N);
  uint8_t* base = static_cast<uint8_t*>(ws);
  double* vals = reinterpret_cast<double*>(base + w.vals);
  double* vals2 = reinterpret_cast<double*>(base + w.vals2);
  double* root = reinterpret_cast<double*>(base + w.root);
  double2* dd = reinterpret_cast<double2*>(base + w.dd);
  double* totals = reinterpret_cast<double*>(base + w.totals);
  int32_t* flag = reinterpret_cast<int32_t*>(base + w.flag);
  double* ckpt = reinterpret_cast<double*>(base + w.ckpt);
  if (!p.valid || p.rdepth > kNodeLevels) return cudaErrorInvalidValue;
  dim3 g1((unsigned)((int64_t)1 << p.t1), (unsigned)B);
  k_pp_node<<<g1, 256, 0, s>>>(m, N, N, p.t1, p.rdepth, halted, j, p.t1 == 0 ? root : vals, dd);
  // fold the complete tree above t1 in tiers of <= 12 levels
  const double* in = vals;
  for (size_t k = 0; k < p.tiers.size(); ++k) {
    const int t_in = p.tiers[k];
    const int t_out = std::max(0, t_in - kTierLevels);
    double* out = t_out == 0 ? root : ((k & 1) ? vals : vals2);
    dim3 g((unsigned)((int64_t)1 << t_out), (unsigned)B);
    k_pp_tier<<<g, 256, 0, s>>>(in, t_in, out, t_out, halted, j);
    in = out;
  }
  const int fe = force_exact_env() ? 1 : 0;
  k_pp_select<<<(unsigned)B, 1024, 0, s>>>(m, N, N, p.t1, root, dd, u, K, j, idx, halted, flag,
                                           totals, fe);
  if (exact_serial_env()) {  // FK_PP_EXACT_SERIAL=1: the one-thread chain (A/B)
    k_pp_exact<<<(unsigned)B, 256, 0, s>>>(m, N, N, u, K, j, idx, halted, flag, totals, ckpt,
                                           w.ntiles);
  } else {
    double* pbuf = reinterpret_cast<double*>(base + w.p);
    double2* tsum = reinterpret_cast<double2*>(base + w.tsum);
    int* epred = reinterpret_cast<int*>(base + w.epred);
    RFun* fun = reinterpret_cast<RFun*>(base + w.fun);
    unsigned int* counters = reinterpret_cast<unsigned int*>(base + w.counters);
    dim3 gt((unsigned)w.ntiles, (unsigned)B);
    // per-batch counters: [2b] for k_ex_tiles, [2b+1] for k_ex_funcs (strided by 2)
    k_ex_tiles<<<gt, kExThreads, 0, s>>>(m, N, halted, flag, totals, j, pbuf, tsum, epred,
                                         counters);
    k_ex_funcs<<<gt, kExThreads, 0, s>>>(pbuf, N, u, K, j, idx, halted, flag, epred, fun, ckpt,
                                         counters + 1);
  }
  return cudaGetLastError();
}

cudaError_t launch_kmeanspp(int dt, const void* X, int64_t B, int64_t N, int64_t d, int64_t K,
                            const double* u, int64_t* idx, int32_t* halted, double* m, void* ws,
                            cudaStream_t s) {
  cudaError_t e = launch_kmeanspp_init(halted, ws, B, N, K, s);
  if (e != cudaSuccess) return e;
  // pruned sweeps need aligned 16-byte rows and a staged row within 200 KB
  const size_t es = dt == DT_F32 ? 4 : dt == DT_F64 ? 8 : 2;
  const size_t rb = (size_t)d * es;
  const bool prune = prune_env() && rb % 16 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                     ((d * 8 + 15) & ~15) + 128 * (rb + 16) <= 200 * 1024;
  uint8_t* extra = static_cast<uint8_t*>(ws) + ws_layout(B, N).bytes;
  int32_t* nearest = reinterpret_cast<int32_t*>(extra);
  double* centers = reinterpret_cast<double*>(extra + al256((size_t)B * N * 4));
  double* cdist =
      reinterpret_cast<double*>(extra + al256((size_t)B * N * 4) + al256((size_t)B * K * d * 8));
  for (int64_t j = 1; j < K; ++j) {
    if (prune) {
      const int64_t jc = j - 1;  // the center this draw's sweep adds
      const int wpb = 8;
      dim3 g((unsigned)std::max<int64_t>(1, (jc + wpb - 1) / wpb), (unsigned)B);
      k_pp_cdist<<<g, 32 * wpb, ((size_t)d * 8 + 15) & ~size_t(15), s>>>(
          X, dt, N, (int)d, idx, K, jc, centers, cdist, halted, j);
      e = sweep_pruned(dt, X, B, N, (int)d, idx, K, jc, m, nearest, cdist, j == 1 ? 1 : 0, halted, j,
                       s);
    } else {
      e = sweep_dispatch(dt, X, B, N, (int)d, N * d, X, N * d, idx, K, j - 1, m, N, j == 1 ? 1 : 0,
                         halted, j, s);
    }
    if (e != cudaSuccess) return e;
    e = launch_kmeanspp_select(m, B, N, u, K, j, idx, halted, ws, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

FK_MODULE_ANCHOR(kmeanspp)

}  // namespace fk
