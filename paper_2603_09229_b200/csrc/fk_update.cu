// fk_update.cu -- sort-inverse centroid update, normalize and objective.
//
// Replaces sort_inverse_update (reference sort_inverse.py:106-149, kernels
// counting_sort / segment_stats / merge_segments _kernels.py:118-171) with a
// contention-free GPU scheme: no per-point scatter into shared accumulators.
//
//   k_hist     histogram of composite keys (b*K + id), smem-privatized when
//              B*K fits in shared memory                      -> counts (exact)
//   k_scan     one-block exclusive scan -> segment offsets, insertion cursors,
//              int64 counts and the reference's synchronized_merges count
//   k_scatter  bucket point indices by key (warp-aggregated cursor bumps);
//              X itself is never permuted (sort_inverse.py:12-13)
//   k_segsum   equal slices of the sorted order per warp; each warp streams the
//              gathered rows with 16-byte vector loads, keeps per-lane running
//              sums, and emits ONE merge per segment: segments owned by the
//              slice are written directly, the <= 2 boundary segments per
//              slice are merged with an f64 reduction.
//
// sums are f64 and counts int64, the reference's ClusterStats dtypes
// (core.py:203-233).  bf16/fp16 rows accumulate in fp32 inside a slice; f32
// and f64 rows accumulate in f64 so fp32 data reproduces the reference's
// sums exactly.
#include <cooperative_groups.h>
#include <stdlib.h>

#include "fk_common.cuh"
#include "fk_kernels.h"

namespace cg = cooperative_groups;

namespace fk {

constexpr int HIST_SMEM_KEYS = 12288;  // 48 KB of int32 bins

FK_DEV double as_f64(float v) { return (double)v; }
FK_DEV double as_f64(double v) { return v; }
FK_DEV double as_f64(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
FK_DEV double as_f64(__half v) { return (double)__half2float(v); }

// ----------------------------------------------------------------- hist
// Each block owns a contiguous range of one batch element's points.  With
// K <= HIST_SMEM_KEYS the block histograms in shared memory and publishes one
// atomic per non-empty bin; otherwise identical keys are warp-aggregated.
// Blocks are laid out per batch element (gridDim.x = B * bpb): block j of
// element b owns a contiguous slice of that element's points, so a shared
// histogram needs only K bins, whatever B is.
__device__ __forceinline__ void range_of(int64_t N, int bpb, int64_t& b, int64_t& lo,
                                         int64_t& hi) {
  b = blockIdx.x / bpb;
  const int j = blockIdx.x - (int)b * bpb;
  const int64_t per = (N + bpb - 1) / bpb;
  lo = b * N + (int64_t)j * per;
  const int64_t end = (int64_t)j * per + per < N ? (int64_t)j * per + per : N;
  hi = b * N + end;
}

// Visit ids[lo, hi) as f(index, id): a scalar head up to 16-byte alignment,
// then int4 loads two at a time (8 ids in flight per thread, so the loop is
// not bound by one load's latency), then a scalar tail.
template <typename F>
__device__ __forceinline__ void for_each_id(const int32_t* __restrict__ ids, int64_t lo,
                                            int64_t hi, F&& f) {
  const int64_t t = threadIdx.x, nt = blockDim.x;
  int64_t a = lo + (int64_t)(((16u - ((uint32_t)(uintptr_t)(ids + lo) & 15u)) & 15u) >> 2);
  if (a > hi) a = hi;
  for (int64_t i = lo + t; i < a; i += nt) f(i, __ldg(ids + i));
  const int64_t nv = (hi - a) >> 2;
  const int4* v = reinterpret_cast<const int4*>(ids + a);
  int64_t q = t;
  for (; q + nt < nv; q += 2 * nt) {
    const int4 w0 = __ldg(v + q), w1 = __ldg(v + q + nt);
    const int64_t i0 = a + 4 * q, i1 = a + 4 * (q + nt);
    f(i0, w0.x);
    f(i0 + 1, w0.y);
    f(i0 + 2, w0.z);
    f(i0 + 3, w0.w);
    f(i1, w1.x);
    f(i1 + 1, w1.y);
    f(i1 + 2, w1.z);
    f(i1 + 3, w1.w);
  }
  for (; q < nv; q += nt) {
    const int4 w0 = __ldg(v + q);
    const int64_t i0 = a + 4 * q;
    f(i0, w0.x);
    f(i0 + 1, w0.y);
    f(i0 + 2, w0.z);
    f(i0 + 3, w0.w);
  }
  for (int64_t i = a + 4 * nv + t; i < hi; i += nt) f(i, __ldg(ids + i));
}

// zero_sums (non-accumulating updates): the blocks also clear the f64 sums
// for k_segsum, a grid-strided slice each, instead of a separate memset.
__global__ void __launch_bounds__(1024) k_hist(const int32_t* __restrict__ ids, int64_t B, int64_t N,
                                               int64_t K, int bpb, int32_t* __restrict__ hist,
                                               int32_t* __restrict__ table,
                                               double* __restrict__ zero_sums, int64_t zero_n) {
  extern __shared__ int32_t sh[];
  if (zero_sums) {
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    const int64_t n2 = zero_n >> 1;  // 16-byte stores when the (caller-owned) buffer allows
    double2* z2 = reinterpret_cast<double2*>(zero_sums);
    if ((reinterpret_cast<uintptr_t>(zero_sums) & 15) == 0) {
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += nt)
        z2[i] = make_double2(0.0, 0.0);
      if ((zero_n & 1) && blockIdx.x == 0 && threadIdx.x == 0) zero_sums[zero_n - 1] = 0.0;
    } else {
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < zero_n; i += nt)
        zero_sums[i] = 0.0;
    }
  }
  const bool use_smem = K <= HIST_SMEM_KEYS;
  int64_t b, lo, hi;
  range_of(N, bpb, b, lo, hi);
  if (use_smem) {
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) sh[k] = 0;
    __syncthreads();
  }
  for_each_id(ids, lo, hi, [&](int64_t, int32_t id) {
    if (id < 0 || id >= K) return;  // validated on the host side
    if (use_smem) {
      atomicAdd(&sh[id], 1);
    } else {
      const int64_t key = b * K + id;
      const unsigned peers = __match_any_sync(__activemask(), key);
      const int leader = __ffs(peers) - 1;
      if ((int)(threadIdx.x & 31) == leader) atomicAdd(&hist[key], __popc(peers));
    }
  });
  if (use_smem) {
    __syncthreads();
    int32_t* trow = table + (int64_t)blockIdx.x * K;  // this block's histogram, reused by the scatter
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
      const int32_t c = sh[k];
      trow[k] = c;
      if (c) atomicAdd(&hist[b * K + k], c);
    }
  }
}

// ----------------------------------------------------------------- scan
// One block of 1024 threads per batch element b.  The block first reduces the
// histogram of all earlier batch elements (its base offset; b*N when every id
// is valid), then walks its own K keys in tiles of 4096 (4 consecutive keys
// per thread, so K <= 4096 is one pass): block-wide exclusive scan per tile
// plus a running carry.  Also produces the int64 counts and the reference's
// synchronized_merges count.
__global__ void __launch_bounds__(1024)
    k_scan(const int32_t* __restrict__ hist, int64_t B, int64_t N, int64_t K, int64_t chunk,
           int accumulate, int64_t* __restrict__ off, int32_t* __restrict__ cursor,
           int64_t* __restrict__ counts, int64_t* __restrict__ merges) {
  __shared__ int64_t warp_tot[32];
  __shared__ unsigned long long warp_mg[32];
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x;
  const int lane = t & 31, w = t >> 5;
  int64_t part = 0;
  for (int64_t i = t; i < b * K; i += 1024) part += hist[i];
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) warp_tot[w] = part;
  __syncthreads();
  int64_t carry = 0;
  for (int i = 0; i < 32; ++i) carry += warp_tot[i];
  __syncthreads();
  unsigned long long mg = 0;
  const uint32_t ch = (uint32_t)chunk;
  // tiles of 4096 keys, 4 consecutive keys per thread: one pass when K <= 4096
  for (int64_t base = 0; base < K; base += 4096) {
    int64_t c[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t kk = base + 4 * t + q;
      c[q] = kk < K ? hist[b * K + kk] : 0;
      sum += c[q];
    }
    int64_t v = sum;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) warp_tot[w] = v;
    __syncthreads();
    if (w == 0) {
      int64_t x = warp_tot[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += u;
      }
      warp_tot[lane] = x;  // inclusive over warps
    }
    __syncthreads();
    int64_t run = carry + v - sum + (w > 0 ? warp_tot[w - 1] : 0);  // exclusive prefix
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t kk = base + 4 * t + q;
      if (kk < K) {
        const int64_t k = b * K + kk;
        off[k] = run;
        cursor[k] = (int32_t)run;
        counts[k] = accumulate ? counts[k] + c[q] : c[q];
        if (c[q] > 0 && merges) {
          // reference merges: the run [s, e) of this key inside its batch element
          // meets floor((e-1)/chunk) - floor(s/chunk) + 1 update chunks
          // (all quantities < 2^31: 32-bit divisions)
          const uint32_t s0 = (uint32_t)(run - b * N), e = s0 + (uint32_t)c[q];
          mg += (unsigned long long)((e - 1) / ch - s0 / ch + 1);
        }
      }
      run += c[q];
    }
    carry += warp_tot[31];
    __syncthreads();
  }
  if (b == B - 1 && t == 0) off[B * K] = carry;
  for (int o = 16; o; o >>= 1) mg += __shfl_xor_sync(0xffffffffu, mg, o);
  if (lane == 0) warp_mg[w] = mg;
  __syncthreads();
  if (w == 0 && merges) {
    unsigned long long m = warp_mg[lane];
    for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    if (lane == 0) atomicAdd((unsigned long long*)merges, m);
  }
}

// ----------------------------------------------------------------- scatter
// Bucket point indices by key.  Block-aggregated: a block histograms its
// contiguous point range in shared memory, reserves ONE contiguous range per
// non-empty key with a single global atomic, then hands out positions with
// shared-memory cursors -- no per-point global atomics, no dependency chains.
__global__ void __launch_bounds__(1024)
    k_scatter_block(const int32_t* __restrict__ ids, int64_t B, int64_t N, int64_t K, int bpb,
                    const int32_t* __restrict__ table, int32_t* __restrict__ cursor,
                    int32_t* __restrict__ order) {
  extern __shared__ int32_t sh[];
  int64_t b, lo, hi;
  range_of(N, bpb, b, lo, hi);
  // this block's histogram (built by k_hist over the same point range):
  // reserve one contiguous range per non-empty key
  const int32_t* trow = table + (int64_t)blockIdx.x * K;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const int32_t c = trow[k];
    sh[k] = c ? atomicAdd(&cursor[b * K + k], c) : 0;
  }
  __syncthreads();
  for_each_id(ids, lo, hi, [&](int64_t i, int32_t id) {
    if (id < 0 || id >= K) return;
    const int pos = atomicAdd(&sh[id], 1);
    order[pos] = (int32_t)i;
  });
}

// Staged variant (K <= SC_KMAX): the block's range is processed in sub-tiles
// of SC_S points.  Each sub-tile is counting-sorted by key in shared memory
// (local ranks from shared atomics, a block scan of the K counts) and then
// written out in sorted order, so consecutive threads store consecutive
// positions of the same key's run: one store instruction touches a few
// 32-byte sectors instead of 32 scattered ones.  Staged entries pack
// (local index << 14) | key into 32 bits.
#ifndef FK_SC_PT
#define FK_SC_PT 16
#endif
constexpr int SC_PT = FK_SC_PT;      // points per thread per sub-tile
constexpr int SC_S = 1024 * SC_PT;   // points per sub-tile
#ifndef FK_SC_MIN_RANGE
#define FK_SC_MIN_RANGE 6144
#endif
constexpr int SC_MIN_RANGE = FK_SC_MIN_RANGE;  // staged only for block ranges at least this long
constexpr int SC_KMAX = 4096;  // keys: 3 K-int tables + the stage fit twice per SM
__global__ void __launch_bounds__(1024, SC_PT <= 8 ? 2 : 1)
    k_scatter_staged(const int32_t* __restrict__ ids, int64_t B, int64_t N, int64_t K, int bpb,
                     const int32_t* __restrict__ table, int32_t* __restrict__ cursor,
                     int32_t* __restrict__ order) {
  extern __shared__ int32_t sm[];
  __shared__ int32_t wtot[32];
  int32_t* gcur = sm;          // next global position of each key for this block
  int32_t* lcnt = sm + K;      // sub-tile counts per key
  int32_t* lbase = sm + 2 * K;  // exclusive scan of lcnt
  uint32_t* stage = reinterpret_cast<uint32_t*>(sm + 3 * K);
  int64_t b, lo, hi;
  range_of(N, bpb, b, lo, hi);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int32_t* trow = table + (int64_t)blockIdx.x * K;
  for (int k = t; k < K; k += 1024) {
    const int32_t c = trow[k];
    gcur[k] = c ? atomicAdd(&cursor[b * K + k], c) : 0;
  }
  for (int64_t s0 = lo; s0 < hi; s0 += SC_S) {
    const int n = (int)(hi - s0 < SC_S ? hi - s0 : SC_S);
    for (int k = t; k < K; k += 1024) lcnt[k] = 0;
    __syncthreads();
    int32_t id[SC_PT], rk[SC_PT];
#pragma unroll
    for (int j = 0; j < SC_PT; ++j) id[j] = t + 1024 * j < n ? __ldg(ids + s0 + t + 1024 * j) : -1;
#pragma unroll
    for (int j = 0; j < SC_PT; ++j) rk[j] = (id[j] >= 0 && id[j] < K) ? atomicAdd(&lcnt[id[j]], 1) : -1;
    __syncthreads();
    // exclusive scan of lcnt: 4 consecutive keys per thread (K <= 4096)
    int v[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = 4 * t + q;
      v[q] = k < K ? lcnt[k] : 0;
      sum += v[q];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wtot[w] = incl;
    __syncthreads();
    if (w == 0) {
      int x = wtot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += u;
      }
      wtot[lane] = x;
    }
    __syncthreads();
    int run = incl - sum + (w ? wtot[w - 1] : 0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = 4 * t + q;
      if (k < K) lbase[k] = run;
      run += v[q];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < SC_PT; ++j)
      if (rk[j] >= 0) stage[lbase[id[j]] + rk[j]] = ((uint32_t)(t + 1024 * j) << 14) | (uint32_t)id[j];
    __syncthreads();
    const int tot = wtot[31];
    for (int p = t; p < tot; p += 1024) {
      const uint32_t e = stage[p];
      const int key = (int)(e & 0x3fffu);
      order[gcur[key] + p - lbase[key]] = (int32_t)(s0 + (e >> 14));
    }
    __syncthreads();
    for (int k = t; k < K; k += 1024) gcur[k] += lcnt[k];
  }
}

// Large B*K: warp-aggregated cursor bumps straight in global memory.
__global__ void k_scatter(const int32_t* __restrict__ ids, int64_t B, int64_t N, int64_t K,
                          int32_t* __restrict__ cursor, int32_t* __restrict__ order) {
  const int64_t P = B * N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += stride) {
    const int64_t b = i / N;
    const int32_t id = ids[i];
    if (id < 0 || id >= K) continue;
    const int64_t key = b * K + id;
    const unsigned mask = __activemask();
    const unsigned peers = __match_any_sync(mask, key);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&cursor[key], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    const int rank = __popc(peers & ((1u << lane) - 1));
    order[base + rank] = (int32_t)i;
  }
}

// ----------------------------------------------------------------- segsum
template <typename T>
struct VecCvt;
template <>
struct VecCvt<__nv_bfloat16> {
  static constexpr int E = 8;
  template <typename A>
  FK_DEV static void add(A* acc, const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[2 * i] += (A)__uint_as_float(w[i] << 16);
      acc[2 * i + 1] += (A)__uint_as_float(w[i] & 0xffff0000u);
    }
  }
};
template <>
struct VecCvt<__half> {
  static constexpr int E = 8;
  template <typename A>
  FK_DEV static void add(A* acc, const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      acc[2 * i] += (A)f.x;
      acc[2 * i + 1] += (A)f.y;
    }
  }
};
template <>
struct VecCvt<float> {
  static constexpr int E = 4;
  template <typename A>
  FK_DEV static void add(A* acc, const uint4& v) {
    acc[0] += (A)__uint_as_float(v.x);
    acc[1] += (A)__uint_as_float(v.y);
    acc[2] += (A)__uint_as_float(v.z);
    acc[3] += (A)__uint_as_float(v.w);
  }
};
template <>
struct VecCvt<double> {
  static constexpr int E = 2;
  template <typename A>
  FK_DEV static void add(A* acc, const uint4& v) {
    acc[0] += __hiloint2double((int)v.y, (int)v.x);
    acc[1] += __hiloint2double((int)v.w, (int)v.z);
  }
};

FK_DEV uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// LPR lanes cover one row with VPL 16-byte vectors each; RPW = 32/LPR rows per
// warp step; U steps are issued back to back to keep bytes in flight.
template <typename T, typename A, int LPR, int VPL, int U>
__global__ void __launch_bounds__(256)
    k_segsum(const T* __restrict__ X, const int32_t* __restrict__ order,
             const int64_t* __restrict__ off, int64_t BK, int64_t P, int64_t L, int64_t d,
             double* __restrict__ sums, const int32_t* __restrict__ ids, int64_t N, int64_t K) {
  constexpr int E = VecCvt<T>::E;
  constexpr int RPW = 32 / LPR;
  constexpr int NA = VPL * E;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, sl = lane % LPR;
  const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t p0 = wg * L;
  if (p0 >= P) return;
  const int64_t p1 = (p0 + L < P) ? p0 + L : P;
  // segment containing p0 (largest key with off[key] <= p0 < off[key+1]) is
  // the key of the point sorted to p0: two dependent loads instead of a
  // log2(BK)-step binary search over off[]
  const int32_t pt = order[p0];
  const int64_t pb = pt / N;
  int64_t key = pb * K + ids[pt];
  if (key < 0 || key >= BK || off[key] > p0 || off[key + 1] <= p0) {
    int64_t lo = 0, hi = BK;  // defensive (ids are validated by the caller)
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (off[mid] <= p0) lo = mid; else hi = mid;
    }
    key = lo;
  }
  int64_t seg_lo = off[key], seg_end = off[key + 1];
  A acc[NA];
#pragma unroll
  for (int e = 0; e < NA; ++e) acc[e] = (A)0;
  const int64_t row_elems = d;
  int64_t p = p0;
  while (p < p1) {
    const int64_t lim = seg_end < p1 ? seg_end : p1;
    if (p + RPW * U <= lim) {
      // software pipeline: the sorted-order indices of the next group are
      // fetched while this group's gathered rows are in flight
      int32_t ri[U];
#pragma unroll
      for (int u = 0; u < U; ++u) ri[u] = __ldg(order + p + u * RPW + sub);
      while (true) {
        uint4 v[U][VPL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const T* rp = X + (int64_t)ri[u] * row_elems;
#pragma unroll
          for (int q = 0; q < VPL; ++q) v[u][q] = ldg_stream(rp + (q * LPR + sl) * E);
        }
        const int64_t pn = p + RPW * U;
        const bool more = pn + RPW * U <= lim;
        if (more) {
#pragma unroll
          for (int u = 0; u < U; ++u) ri[u] = __ldg(order + pn + u * RPW + sub);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < VPL; ++q) VecCvt<T>::add(acc + q * E, v[u][q]);
        p = pn;
        if (!more) break;
      }
    }
    // tail of the segment (< RPW*U rows): same batched gathers, masked per row
    if (p < lim) {
      int32_t ri[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = p + u * RPW + sub;
        ri[u] = r < lim ? __ldg(order + r) : -1;
      }
      uint4 v[U][VPL];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const T* rp = X + (int64_t)(ri[u] < 0 ? 0 : ri[u]) * row_elems;
#pragma unroll
        for (int q = 0; q < VPL; ++q)
          v[u][q] = ri[u] >= 0 ? ldg_stream(rp + (q * LPR + sl) * E) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < VPL; ++q) VecCvt<T>::add(acc + q * E, v[u][q]);
    }
    p = lim;
    // flush this segment's partial (one merge per segment)
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
      for (int e = 0; e < NA; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    if (sub == 0) {
      const bool owned = seg_lo >= p0 && seg_end <= p1;
      double* dst = sums + key * d;
#pragma unroll
      for (int q = 0; q < VPL; ++q)
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int64_t j = (int64_t)(q * LPR + sl) * E + e;
          if (owned)
            dst[j] += (double)acc[q * E + e];
          else
            atomicAdd(dst + j, (double)acc[q * E + e]);
        }
    }
#pragma unroll
    for (int e = 0; e < NA; ++e) acc[e] = (A)0;
    if (p < p1) {
      // next non-empty segment
      ++key;
      while (off[key + 1] <= p) ++key;
      seg_lo = off[key];
      seg_end = off[key + 1];
    }
  }
}

// Any row width: one warp per slice, lanes stride over the features.
template <typename T>
__global__ void k_segsum_generic(const T* __restrict__ X, const int32_t* __restrict__ order,
                                 const int64_t* __restrict__ off, int64_t BK, int64_t P,
                                 int64_t L, int64_t d, double* __restrict__ sums) {
  const int lane = threadIdx.x & 31;
  const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t p0 = wg * L;
  if (p0 >= P) return;
  const int64_t p1 = (p0 + L < P) ? p0 + L : P;
  int64_t lo = 0, hi = BK;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (off[mid] <= p0) lo = mid; else hi = mid;
  }
  int64_t key = lo;
  int64_t p = p0;
  while (p < p1) {
    const int64_t seg_lo = off[key], seg_end = off[key + 1];
    const int64_t lim = seg_end < p1 ? seg_end : p1;
    const bool owned = seg_lo >= p0 && seg_end <= p1;
    for (int64_t j0 = 0; j0 < d; j0 += 32) {
      const int64_t j = j0 + lane;
      double acc = 0.0;
      if (j < d)
        for (int64_t r = p; r < lim; ++r) acc += as_f64(X[(int64_t)order[r] * d + j]);
      if (j < d) {
        if (owned)
          sums[key * d + j] += acc;
        else
          atomicAdd(sums + key * d + j, acc);
      }
    }
    p = lim;
    if (p < p1) {
      ++key;
      while (off[key + 1] <= p) ++key;
    }
  }
}

// Blocks per batch element for the histogram / scatter passes: ~2 waves in
// total, each block owning >= 8192 points so the per-block K-bin table, its
// scan and its cursor reservations amortize (same-box A/B,
// profiles/r01_ab_update_bpb.txt: 2048 -> 8192 points took config 2 from 73
// to 69 us and config 4 from 63 to 57 us; config 3 is capped by the wave count).
static int64_t update_bpb(int64_t B, int64_t N, int num_sms) {
  static int64_t min_range = -1;  // FK_UPDATE_MIN_RANGE: points per block lower bound (A/B)
  if (min_range < 0) {
    const char* e = getenv("FK_UPDATE_MIN_RANGE");
    min_range = e ? atoll(e) : 8192;
    if (min_range < 2048) min_range = 2048;  // the workspace table is sized for >= 2048
  }
  int64_t bpb = ((int64_t)num_sms * 2 + B - 1) / B;
  const int64_t max_bpb = (N + min_range - 1) / min_range;
  if (bpb > max_bpb) bpb = max_bpb;
  return bpb < 1 ? 1 : bpb;
}
constexpr int kMaxSms = 256;  // workspace bound for any sm_100 part

// ------------------------------------------------- one-kernel cluster update
// Small per-batch problems (config 4: B=64 x N=16k, K=256, d=64, fp16): one
// thread-block cluster of C CTAs per batch element does the whole update in
// shared memory, with no global scratch and one launch:
//   1. each CTA histograms its N/C ids (shared bins) and counting-sorts its
//      local point indices by id (shared cursors);
//   2. rank 0 reads every CTA's bins over DSMEM: exact int64 counts and the
//      reference's synchronized_merges count for this batch element;
//   3. each CTA walks its local sorted order in contiguous runs per lane
//      group, gathers the rows (16-B vectors), keeps fp32 running sums and
//      merges ONCE per (run, segment) into its shared K x d fp32 table;
//   4. CTA r reduces key range r of the C tables over DSMEM in fixed rank
//      order and stores f64 sums directly (no global atomics).
constexpr int CU_THREADS = 256;
constexpr int CU_PMAX = 8192;               // local points per CTA
constexpr size_t CU_TABLE_MAX = 96 * 1024;  // K * d * 4 bytes of shared sums

template <typename T>
__global__ void __launch_bounds__(CU_THREADS)
    k_update_cluster(const T* __restrict__ X, const int32_t* __restrict__ ids, int64_t N, int K,
                     int d, int64_t chunk, int accumulate, double* __restrict__ sums,
                     int64_t* __restrict__ counts, int64_t* __restrict__ merges) {
  extern __shared__ __align__(16) uint8_t cu_sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int r = (int)cluster.block_rank();
  const int64_t b = blockIdx.x / C;
  const int64_t per = (N + C - 1) / C;
  const int64_t lo = (int64_t)r * per;
  const int64_t hi = lo + per < N ? lo + per : N;
  const int np = hi > lo ? (int)(hi - lo) : 0;
  float* table = reinterpret_cast<float*>(cu_sm);                         // K*d
  int32_t* hist = reinterpret_cast<int32_t*>(cu_sm + (size_t)K * d * 4);  // K
  int32_t* cur = hist + K;                                                // K
  int32_t* order = cur + K;                                               // per
  int32_t* sid = order + per;                                             // per: local ids
  __shared__ unsigned long long s_mg;
  __shared__ int64_t wtot[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int k = t; k < K; k += CU_THREADS) hist[k] = 0;
  for (int e = t; e < K * d; e += CU_THREADS) table[e] = 0.f;
  if (t == 0) s_mg = 0;
  __syncthreads();
  const int32_t* idb = ids + b * N + lo;
  for (int i = t; i < np; i += CU_THREADS) {
    const int32_t id = __ldg(idb + i);
    sid[i] = id;
    if (id >= 0 && id < K) atomicAdd(&hist[id], 1);
  }
  __syncthreads();
  // local exclusive scan of the bins -> cursors (one warp per 32-key tile, serial carry)
  if (warp == 0) {
    int carry = 0;
    for (int base = 0; base < K; base += 32) {
      const int k = base + lane;
      const int c = k < K ? hist[k] : 0;
      int v = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (k < K) cur[k] = carry + v - c;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  cluster.sync();  // every CTA's bins are final (read remotely below)
  if (r == 0) {
    // exact counts + the reference's merge count for this batch element
    int64_t carry = 0;
    unsigned long long mg = 0;
    const uint32_t ch = (uint32_t)chunk;
    for (int base = 0; base < K; base += CU_THREADS) {
      const int k = base + t;
      int64_t c = 0;
      if (k < K)
        for (int q = 0; q < C; ++q) c += *cluster.map_shared_rank(hist + k, q);
      int64_t v = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane == 31) wtot[warp] = v;
      __syncthreads();
      int64_t wbase = 0;
      for (int w = 0; w < warp; ++w) wbase += wtot[w];
      const int64_t run = carry + wbase + v - c;
      if (k < K) {
        counts[b * K + k] = accumulate ? counts[b * K + k] + c : c;
        if (c > 0) {
          const uint32_t s0 = (uint32_t)run, e = s0 + (uint32_t)c;
          mg += (unsigned long long)((e - 1) / ch - s0 / ch + 1);
        }
      }
      int64_t tot = 0;
      for (int w = 0; w < CU_THREADS / 32; ++w) tot += wtot[w];
      carry += tot;
      __syncthreads();
    }
    for (int o = 16; o; o >>= 1) mg += __shfl_xor_sync(0xffffffffu, mg, o);
    if (lane == 0 && mg) atomicAdd(&s_mg, mg);
  }
  // local counting sort of the point indices (X is never permuted)
  for (int i = t; i < np; i += CU_THREADS) {
    const int32_t id = sid[i];
    if (id >= 0 && id < K) order[atomicAdd(&cur[id], 1)] = i;
  }
  __syncthreads();
  // cur[k] is now the END of key k's local run; the valid sorted length:
  const int nv = K > 0 ? cur[K - 1] : 0;
  // segmented sums: LPR lanes cover one row, each lane group walks a
  // contiguous run of the local sorted order
  constexpr int E = 16 / (int)sizeof(T);
  const int vpr = d / E;                // 16-B vectors per row
  const int lpr = vpr >= 32 ? 32 : vpr; // lanes per row (power of two: d in shape buckets)
  const int vpl = vpr / lpr;            // vectors per lane
  const int groups = CU_THREADS / lpr;
  const int gid = t / lpr, gl = t % lpr;
  const int run = (nv + groups - 1) / groups;
  const int p0 = gid * run, p1 = p0 + run < nv ? p0 + run : nv;
  const T* xb = X + (b * N + lo) * (int64_t)d;
  if (p0 < p1) {
    // key of position p0: first k with cur[k] > p0 (cur = run ends)
    int klo = 0, khi = K - 1;
    while (klo < khi) {
      const int mid = (klo + khi) >> 1;
      if (cur[mid] > p0) khi = mid; else klo = mid + 1;
    }
    for (int v0 = 0; v0 < vpl; ++v0) {
      const int col = (v0 * lpr + gl) * E;
      float acc[E];
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = 0.f;
      int k = klo, ke = cur[klo], nrow = 0;
      auto flush = [&]() {
        if (nrow) {
          float* dst = table + (size_t)k * d + col;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            atomicAdd(dst + e, acc[e]);
            acc[e] = 0.f;
          }
          nrow = 0;
        }
      };
      // CU_U gathers in flight across segment boundaries, added in sorted order;
      // one merge per (run, segment)
      constexpr int CU_U = 16;
      for (int p = p0; p < p1; p += CU_U) {
        const int n = p1 - p < CU_U ? p1 - p : CU_U;
        uint4 v[CU_U];
#pragma unroll
        for (int u = 0; u < CU_U; ++u)
          if (u < n) v[u] = ldg_stream(xb + (int64_t)order[p + u] * d + col);
#pragma unroll
        for (int u = 0; u < CU_U; ++u) {
          if (u < n) {
            while (p + u >= ke) {  // segment boundary (skipping empty keys)
              flush();
              ++k;
              ke = cur[k];
            }
            VecCvt<T>::add(acc, v[u]);
            ++nrow;
          }
        }
      }
      flush();
    }
  }
  cluster.sync();  // every table complete
  // CTA r reduces keys [r*K/C, (r+1)*K/C) across the cluster, fixed rank order
  const int k0 = (int)((int64_t)K * r / C), k1 = (int)((int64_t)K * (r + 1) / C);
  const float* rt[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) rt[q] = cluster.map_shared_rank(table, q < C ? q : 0);
  for (int e = k0 * d + t; e < k1 * d; e += CU_THREADS) {
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = q < C ? rt[q][e] : 0.f;  // all remote loads in flight
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < C) acc += (double)v[q];
    double* o = sums + b * (int64_t)K * d + e;
    *o = accumulate ? *o + acc : acc;
  }
  if (r == 0 && t == 0 && merges && s_mg) atomicAdd((unsigned long long*)merges, s_mg);
  cluster.sync();  // keep every table alive until all remote reads are done
}

// cluster size for the one-kernel path, or 0 when it does not apply
static int cluster_update_size(int dt, int64_t B, int64_t N, int64_t K, int64_t d, int num_sms) {
  // Opt-in only (FK_UPDATE_CLUSTER=1): same-box A/B at config 4 measured 66.9 us
  // against 61.4 us for the four-kernel path (0.45 waves of 8-warp CTAs and
  // serialized phases leave HBM at 24%; profiles/r01_ab_cluster.txt).
  const char* e = getenv("FK_UPDATE_CLUSTER");
  if (!(e && e[0] == '1')) return 0;
  if (dt != DT_BF16 && dt != DT_F16) return 0;  // f32/f64 keep f64 accumulation (bitwise path)
  if ((d * 2) % 16 != 0 || d > 256 || (d / 8 & (d / 8 - 1)) != 0) return 0;
  if ((size_t)K * d * 4 > CU_TABLE_MAX || K > 8192) return 0;
  for (int C = 1; C <= 8; C <<= 1) {
    const int64_t per = (N + C - 1) / C;
    if (per > CU_PMAX) continue;
    // enough CTAs to cover the machine when the batch is small
    if (B * C < num_sms && C < 8 && (N + 2 * C - 1) / (2 * C) >= 512) continue;
    return C;
  }
  return 0;
}

static size_t cluster_update_smem(int64_t N, int64_t K, int64_t d, int C) {
  const int64_t per = (N + C - 1) / C;
  return (size_t)K * d * 4 + (size_t)K * 8 + (size_t)per * 8;
}

template <typename T>
static cudaError_t launch_cluster_update(const void* X, const int32_t* ids, int64_t B, int64_t N,
                                         int64_t K, int64_t d, int64_t chunk, int accumulate,
                                         double* sums, int64_t* counts, int64_t* merges, int C,
                                         cudaStream_t s) {
  const size_t smem = cluster_update_smem(N, K, d, C);
  cudaFuncSetAttribute(k_update_cluster<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(B * C));
  cfg.blockDim = dim3(CU_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_update_cluster<T>, static_cast<const T*>(X), ids, N, (int)K,
                            (int)d, chunk, accumulate, sums, counts, merges);
}

// --------------------------------------------- multi-GPU exchange packing
// The per-iteration all-reduce moves ONE f64 buffer [sums | counts | obj | changed]
// (distributed.py); counts are exact in f64 below 2^53.  One launch each way.
__global__ void k_stats_pack(const int64_t* __restrict__ counts, const double* __restrict__ obj,
                             const int32_t* __restrict__ changed, double* __restrict__ red,
                             int64_t BK, int64_t B) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < BK) red[i] = (double)counts[i];
  else if (i < BK + B) red[i] = obj[i - BK];
  else if (i == BK + B) red[i] = (double)*changed;
}
__global__ void k_stats_unpack(const double* __restrict__ red, int64_t* __restrict__ counts,
                               double* __restrict__ obj, int32_t* __restrict__ changed, int64_t BK,
                               int64_t B) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < BK) counts[i] = (int64_t)red[i];
  else if (i < BK + B) obj[i - BK] = red[i];
  else if (i == BK + B) *changed = red[i] > 0.0 ? 1 : 0;
}
// The reference's synchronized_merges for GLOBAL counts (sharded runs): each
// key's run [s, e) in its batch element's sorted order meets
// floor((e-1)/chunk) - floor(s/chunk) + 1 update chunks (sort_inverse.py:159-165),
// s the exclusive prefix of the counts.  One block walks every batch element
// (B*K is small), so the result is stored, not accumulated.
__global__ void __launch_bounds__(1024)
    k_merges_counts(const int64_t* __restrict__ counts, int64_t B, int64_t K, int64_t chunk,
                    int64_t* __restrict__ merges, int accumulate) {
  __shared__ int64_t wtot[32];
  __shared__ unsigned long long wmg[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  unsigned long long mg = 0;
  for (int64_t b = 0; b < B; ++b) {
    int64_t carry = 0;
    for (int64_t base = 0; base < K; base += 1024) {
      const int64_t k = base + t;
      const int64_t c = k < K ? counts[b * K + k] : 0;
      int64_t v = c;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane == 31) wtot[w] = v;
      __syncthreads();
      int64_t before = 0, tot = 0;
      for (int q = 0; q < 32; ++q) {
        if (q < w) before += wtot[q];
        tot += wtot[q];
      }
      if (c > 0) {
        const int64_t s0 = carry + before + v - c, e = s0 + c;
        mg += (unsigned long long)((e - 1) / chunk - s0 / chunk + 1);
      }
      carry += tot;
      __syncthreads();
    }
  }
  for (int o = 16; o; o >>= 1) mg += __shfl_xor_sync(0xffffffffu, mg, o);
  if (lane == 0) wmg[w] = mg;
  __syncthreads();
  if (t == 0) {
    unsigned long long m = 0;
    for (int q = 0; q < 32; ++q) m += wmg[q];
    *merges = accumulate ? *merges + (int64_t)m : (int64_t)m;
  }
}
cudaError_t launch_merges_counts(const int64_t* counts, int64_t B, int64_t K, int64_t chunk,
                                 int64_t* merges, int accumulate, cudaStream_t s) {
  k_merges_counts<<<1, 1024, 0, s>>>(counts, B, K, chunk < 1 ? 1 : chunk, merges, accumulate);
  return cudaGetLastError();
}

cudaError_t launch_stats_pack(int unpack, int64_t* counts, double* obj, int32_t* changed,
                              double* red, int64_t BK, int64_t B, cudaStream_t s) {
  const int64_t n = BK + B + 1;
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (unpack)
    k_stats_unpack<<<grid, 256, 0, s>>>(red, counts, obj, changed, BK, B);
  else
    k_stats_pack<<<grid, 256, 0, s>>>(counts, obj, changed, red, BK, B);
  return cudaGetLastError();
}

size_t update_workspace_bytes(int64_t B, int64_t N, int64_t K) {
  const int64_t BK = B * K, P = B * N;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const int64_t table = K <= HIST_SMEM_KEYS ? B * update_bpb(B, N, kMaxSms) * K : 0;
  return al(BK * 4) + al(BK * 4) + al((BK + 1) * 8) + al(P * 4) + al(table * 4);
}

template <typename T, typename A>
static cudaError_t dispatch_segsum(const void* X, const int32_t* order, const int64_t* off,
                                   int64_t BK, int64_t P, int64_t d, double* sums, int num_sms,
                                   cudaStream_t s, const int32_t* ids, int64_t N, int64_t K) {
  constexpr int E = VecCvt<T>::E;
  const int th = 256;
  // warp slices per SM: 32 (same-box A/B, profiles/r01_ab_segsum.txt: 64 -> 32
  // took config 2 from 67.8 to 64.1 us and config 4 from 52 to 49.5 us, config 3
  // unchanged; 16 starves config 3 of bytes in flight).  FK_SEGSUM_WPS overrides.
  static int wps = -1;
  if (wps < 0) {
    const char* e = getenv("FK_SEGSUM_WPS");
    wps = e ? atoi(e) : 32;
    if (wps < 1) wps = 32;
  }
  const int64_t want_warps = (int64_t)num_sms * wps;
  int64_t L = (P + want_warps - 1) / want_warps;
  if (L < 64) L = 64;
  const int64_t warps = (P + L - 1) / L;
  const unsigned grid = (unsigned)((warps * 32 + th - 1) / th);
  const int64_t row_bytes = d * (int64_t)sizeof(T);
  const bool vec_ok = (row_bytes % 16) == 0;
  const int64_t nvec = row_bytes / 16;  // 16-byte vectors per row
  const T* x = (const T*)X;
#define FK_SEG(LPR, VPL, U) \
  k_segsum<T, A, LPR, VPL, U><<<grid, th, 0, s>>>(x, order, off, BK, P, L, d, sums, ids, N, K)
  if (vec_ok) {
    switch (nvec) {
      case 1: FK_SEG(1, 1, 4); break;
      case 2: FK_SEG(2, 1, 4); break;
      case 4: FK_SEG(4, 1, 4); break;
      case 8: FK_SEG(8, 1, 8); break;
      case 16: FK_SEG(16, 1, 8); break;
      case 32: FK_SEG(32, 1, 4); break;
      case 64: FK_SEG(32, 2, 2); break;
      case 128: FK_SEG(32, 4, 1); break;
      default:
        k_segsum_generic<T><<<grid, th, 0, s>>>(x, order, off, BK, P, L, d, sums);
    }
  } else {
    k_segsum_generic<T><<<grid, th, 0, s>>>(x, order, off, BK, P, L, d, sums);
  }
#undef FK_SEG
  (void)E;
  return cudaGetLastError();
}

cudaError_t launch_update(int dt, const void* X, const int32_t* ids, int64_t B, int64_t N,
                          int64_t K, int64_t d, int64_t chunk, int accumulate, double* sums,
                          int64_t* counts, int64_t* merges, void* ws, int num_sms,
                          cudaStream_t s) {
  const int64_t BK = B * K, P = B * N;
  const int64_t chc = chunk < 1 ? 1 : (chunk > N ? N : chunk);
  if (const int C = cluster_update_size(dt, B, N, K, d, num_sms)) {
    return dt == DT_BF16
               ? launch_cluster_update<__nv_bfloat16>(X, ids, B, N, K, d, chc, accumulate, sums,
                                                      counts, merges, C, s)
               : launch_cluster_update<__half>(X, ids, B, N, K, d, chc, accumulate, sums, counts,
                                               merges, C, s);
  }
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  uint8_t* w = (uint8_t*)ws;
  int32_t* hist = (int32_t*)w;
  w += al(BK * 4);
  int32_t* cursor = (int32_t*)w;
  w += al(BK * 4);
  int64_t* off = (int64_t*)w;
  w += al((BK + 1) * 8);
  int32_t* order = (int32_t*)w;
  w += al(P * 4);
  int32_t* table = (int32_t*)w;  // per-block histograms (shared-histogram path)
  cudaError_t e;
  if ((e = cudaMemsetAsync(hist, 0, BK * 4, s)) != cudaSuccess) return e;
  // sums are cleared inside k_hist (below) unless accumulating
  const int64_t bpb = update_bpb(B, N, num_sms < kMaxSms ? num_sms : kMaxSms);
  const unsigned blocks = (unsigned)(B * bpb);
  const bool smem_keys = K <= HIST_SMEM_KEYS;
  const size_t hsm = smem_keys ? K * 4 : 0;
  k_hist<<<blocks, 1024, hsm, s>>>(ids, B, N, K, (int)bpb, hist, table, accumulate ? nullptr : sums,
                                   BK * d);
  const int64_t ch = chunk < 1 ? 1 : (chunk > N ? N : chunk);
  k_scan<<<(unsigned)B, 1024, 0, s>>>(hist, B, N, K, ch, accumulate, off, cursor, counts, merges);
  static int staged_env = -1;  // FK_UPDATE_SCATTER=block: the unstaged block scatter (A/B)
  if (staged_env < 0) {
    const char* e = getenv("FK_UPDATE_SCATTER");
    staged_env = (e && e[0] == 'b') ? 0 : 1;
  }
  // staged only for block ranges of >= 6K points: shorter ranges pay the
  // per-sub-tile scan and barriers without longer runs (3.5K-point ranges:
  // 72 -> 74 us at config 2, 62 -> 66 us at config 4); with the 8K-point
  // blocks of update_bpb it is 3-4% faster there (profiles/r01_ab_scatter_min_range.txt).
  // update_bpb gives ranges in (4K, 8K] unless the wave cap binds, so the
  // threshold sits inside that interval rather than at its top.
  if (smem_keys && K <= SC_KMAX && staged_env && (N + bpb - 1) / bpb >= SC_MIN_RANGE) {
    const size_t ssm = (3 * K + SC_S) * 4;
    static int attr_dev_mask = 0;  // one-time per device (keeps graph capture free of it)
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_dev_mask & (1 << (dev & 31)))) {
      cudaFuncSetAttribute(k_scatter_staged, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)((3 * SC_KMAX + SC_S) * 4));
      attr_dev_mask |= 1 << (dev & 31);
    }
    k_scatter_staged<<<blocks, 1024, ssm, s>>>(ids, B, N, K, (int)bpb, table, cursor, order);
  } else if (smem_keys)
    k_scatter_block<<<blocks, 1024, hsm, s>>>(ids, B, N, K, (int)bpb, table, cursor, order);
  else
    k_scatter<<<(unsigned)((P + 511) / 512 < num_sms * 4 ? (P + 511) / 512 : num_sms * 4), 512, 0,
                s>>>(ids, B, N, K, cursor, order);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  switch (dt) {
    case DT_BF16: return dispatch_segsum<__nv_bfloat16, float>(X, order, off, BK, P, d, sums, num_sms, s, ids, N, K);
    case DT_F16: return dispatch_segsum<__half, float>(X, order, off, BK, P, d, sums, num_sms, s, ids, N, K);
    case DT_F32: return dispatch_segsum<float, double>(X, order, off, BK, P, d, sums, num_sms, s, ids, N, K);
    default: return dispatch_segsum<double, double>(X, order, off, BK, P, d, sums, num_sms, s, ids, N, K);
  }
}

// ----------------------------------------------------------------- normalize
constexpr int NORM_RW = 4;  // centroid rows per warp in k_normalize

template <typename TM, typename TO>
__global__ void __launch_bounds__(256)
    k_normalize(const double* __restrict__ sums, const int64_t* __restrict__ counts,
                const TM* __restrict__ prev, TM* __restrict__ out, TO* __restrict__ operand,
                uint8_t* __restrict__ empty, double* max_shift2, int64_t BK, int64_t d) {
  __shared__ double wmax[8];
  // NORM_RW rows per warp, every load of a pass (64 columns of each row) issued
  // before the first division so the latencies overlap, and 4x fewer blocks
  // (and shift atomics).  Each element is read and written by the same thread
  // only, so out may alias prev.
  constexpr int RW = NORM_RW, NR = 2;
  const int64_t row0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * RW;
  const int lane = threadIdx.x & 31;
  int64_t cnt[RW];
  double sh[RW];
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    cnt[q] = row0 + q < BK ? counts[row0 + q] : 0;
    sh[q] = 0.0;
  }
  for (int64_t j0 = 0; j0 < d; j0 += 32 * NR) {
    double sv[RW][NR];
    TM pv[RW][NR];
#pragma unroll
    for (int q = 0; q < RW; ++q)
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int64_t j = j0 + lane + 32 * r;
        if (row0 + q < BK && j < d) {
          sv[q][r] = sums[(row0 + q) * d + j];
          pv[q][r] = prev[(row0 + q) * d + j];
        }
      }
#pragma unroll
    for (int q = 0; q < RW; ++q)
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int64_t j = j0 + lane + 32 * r;
        if (row0 + q < BK && j < d) {
          const int64_t o = (row0 + q) * d + j;
          TM nv = pv[q][r];
          if (cnt[q] > 0) nv = (TM)(sv[q][r] / (double)cnt[q]);  // correctly rounded, as numpy
          out[o] = nv;
          if (operand) operand[o] = (TO)(float)nv;
          const double df = (double)nv - (double)pv[q][r];
          sh[q] += df * df;
        }
      }
  }
  if (lane == 0 && empty) {
#pragma unroll
    for (int q = 0; q < RW; ++q)
      if (row0 + q < BK) empty[row0 + q] = cnt[q] > 0 ? 0 : 1;
  }
  if (max_shift2) {
    double m = 0.0;
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      double v = sh[q];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      m = fmax(m, v);
    }
    if (lane == 0) wmax[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      double mb = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mb = fmax(mb, wmax[w]);
      // non-negative doubles order like their bit patterns
      atomicMax((unsigned long long*)max_shift2, (unsigned long long)__double_as_longlong(mb));
    }
  }
}

template <typename TM>
static cudaError_t norm_dispatch(int operand_dt, const double* sums, const int64_t* counts,
                                 const void* prev, void* out, void* operand_out, uint8_t* empty,
                                 double* ms2, int64_t BK, int64_t d, cudaStream_t s) {
  const int th = 256;
  const int64_t rows_per_block = (th / 32) * NORM_RW;
  const unsigned grid = (unsigned)((BK + rows_per_block - 1) / rows_per_block);
  const TM* pv = (const TM*)prev;
  TM* ov = (TM*)out;
  if (!operand_out)
    k_normalize<TM, float><<<grid, th, 0, s>>>(sums, counts, pv, ov, nullptr, empty, ms2, BK, d);
  else if (operand_dt == DT_BF16)
    k_normalize<TM, __nv_bfloat16><<<grid, th, 0, s>>>(sums, counts, pv, ov,
                                                      (__nv_bfloat16*)operand_out, empty, ms2, BK, d);
  else if (operand_dt == DT_F16)
    k_normalize<TM, __half><<<grid, th, 0, s>>>(sums, counts, pv, ov, (__half*)operand_out, empty,
                                               ms2, BK, d);
  else if (operand_dt == DT_F32)
    k_normalize<TM, float><<<grid, th, 0, s>>>(sums, counts, pv, ov, (float*)operand_out, empty,
                                              ms2, BK, d);
  else
    k_normalize<TM, double><<<grid, th, 0, s>>>(sums, counts, pv, ov, (double*)operand_out, empty,
                                               ms2, BK, d);
  return cudaGetLastError();
}

cudaError_t launch_normalize(int master_dt, const double* sums, const int64_t* counts,
                             const void* prev, void* out, int operand_dt, void* operand_out,
                             uint8_t* empty_mask, double* max_shift2, int64_t B, int64_t K,
                             int64_t d, cudaStream_t s) {
  if (master_dt == DT_F64)
    return norm_dispatch<double>(operand_dt, sums, counts, prev, out, operand_out, empty_mask,
                                 max_shift2, B * K, d, s);
  return norm_dispatch<float>(operand_dt, sums, counts, prev, out, operand_out, empty_mask,
                              max_shift2, B * K, d, s);
}

// ----------------------------------------------------------------- objective
// Deterministic two-level reduction (fixed 8192-element blocks, fixed trees).
// For float32 min_dists every float64 partial sum is exact in practice, so
// the result equals numpy's np.sum(m, dtype=float64) bit for bit; for
// float64 data the summation order differs from numpy's pairwise tree.
constexpr int OBJ_BLOCK = 8192;

template <typename T>
__global__ void k_obj_partial(const T* __restrict__ m, int64_t B, int64_t N, int64_t nblk,
                              double* part) {
  __shared__ double red[256];
  const int64_t b = blockIdx.y, blk = blockIdx.x;
  const int64_t lo = blk * OBJ_BLOCK;
  const int64_t hi = (lo + OBJ_BLOCK < N) ? lo + OBJ_BLOCK : N;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += 256) acc += (double)m[b * N + i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[b * nblk + blk] = red[0];
}

__global__ void k_obj_final(const double* part, int64_t B, int64_t nblk, double* out) {
  __shared__ double red[256];
  const int64_t b = blockIdx.x;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < nblk; i += 256) acc += part[b * nblk + i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[b] = red[0];
}

size_t objective_workspace_bytes(int64_t B, int64_t N) {
  return (size_t)(B * ((N + OBJ_BLOCK - 1) / OBJ_BLOCK)) * 8 + 256;
}

cudaError_t launch_objective(int mind_is_f64, const void* mind, int64_t B, int64_t N, double* out,
                             void* ws, cudaStream_t s) {
  const int64_t nblk = (N + OBJ_BLOCK - 1) / OBJ_BLOCK;
  double* part = (double*)ws;
  dim3 grid((unsigned)nblk, (unsigned)B);
  if (mind_is_f64)
    k_obj_partial<double><<<grid, 256, 0, s>>>((const double*)mind, B, N, nblk, part);
  else
    k_obj_partial<float><<<grid, 256, 0, s>>>((const float*)mind, B, N, nblk, part);
  k_obj_final<<<(unsigned)B, 256, 0, s>>>(part, B, nblk, out);
  return cudaGetLastError();
}

// ----------------------------------------------------------------- scatter foil
template <typename T>
__global__ void k_scatter_atomic(const T* __restrict__ X, const int32_t* __restrict__ ids,
                                 int64_t B, int64_t N, int64_t K, int64_t d, double* sums,
                                 int64_t* counts) {
  const int64_t P = B * N;
  const int64_t total = P * d;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t i = e / d, j = e - i * d;
    const int64_t b = i / N;
    const int32_t id = ids[i];
    if (id < 0 || id >= K) continue;
    atomicAdd(&sums[(b * K + id) * d + j], as_f64(X[e]));
    if (j == 0) atomicAdd((unsigned long long*)&counts[b * K + id], 1ull);
  }
}

cudaError_t launch_scatter(int dt, const void* X, const int32_t* ids, int64_t B, int64_t N,
                           int64_t K, int64_t d, double* sums, int64_t* counts, cudaStream_t s) {
  cudaMemsetAsync(sums, 0, B * K * d * 8, s);
  cudaMemsetAsync(counts, 0, B * K * 8, s);
  const unsigned grid = 148 * 8;
  switch (dt) {
    case DT_BF16:
      k_scatter_atomic<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)X, ids, B, N, K,
                                                          d, sums, counts);
      break;
    case DT_F16:
      k_scatter_atomic<__half><<<grid, 256, 0, s>>>((const __half*)X, ids, B, N, K, d, sums, counts);
      break;
    case DT_F32:
      k_scatter_atomic<float><<<grid, 256, 0, s>>>((const float*)X, ids, B, N, K, d, sums, counts);
      break;
    default:
      k_scatter_atomic<double><<<grid, 256, 0, s>>>((const double*)X, ids, B, N, K, d, sums,
                                                    counts);
  }
  return cudaGetLastError();
}

}  // namespace fk
