// fk_update.cu -- sort-inverse centroid update, normalize and objective.
//
// Replaces sort_inverse_update (reference sort_inverse.py:106-149, kernels
// counting_sort / segment_stats / merge_segments _kernels.py:118-171) with a
// contention-free GPU scheme: no per-point scatter into shared accumulators,
// and a result that is bitwise reproducible run to run.
//
//   k_hist       per-block histograms of the cluster ids over contiguous point
//                ranges (shared-memory bins; global rows for very large K)
//   k_colscan    per key: exclusive prefix of the block histograms in block
//                order (each block's base inside the key's run) and the totals
//   k_scan       per batch element: key offsets, int64 counts and the
//                reference's synchronized_merges count
//   k_scatter    each block STABLY sorts its range by id in shared memory
//                (LSD radix passes of <= 8 bits; per-warp digit counters and
//                match.any ranks, no atomics) and writes the point indices at
//                off[key] + block base + rank: the global order is the
//                reference's stable argsort (_kernels.py:118-132); X itself is
//                never permuted (sort_inverse.py:12-13)
//   k_segsum     equal slices of the sorted order per warp; 16-byte row
//                gathers, per-lane running sums, ONE merge per segment: owned
//                segments are stored directly, segments spanning slices leave
//                a partial per slice and the last slice to arrive adds them in
//                slice order (the reference merges in ascending order,
//                _kernels.py:163-171, sort_inverse.py:159-165)
//
// sums are f64 and counts int64, the reference's ClusterStats dtypes
// (core.py:203-233).  bf16/fp16 rows accumulate in fp32 inside a slice; f32
// and f64 rows accumulate in f64.  Every summation order is a fixed function
// of (ids, shape, SM count), so two runs give the same bits.
#include <stdlib.h>

#include "fk_common.cuh"
#include "fk_kernels.h"

namespace fk {

constexpr int HIST_SMEM_KEYS = 12288;  // 48 KB of int32 bins

FK_DEV double as_f64(float v) { return (double)v; }
FK_DEV double as_f64(double v) { return v; }
FK_DEV double as_f64(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
FK_DEV double as_f64(__half v) { return (double)__half2float(v); }

// ----------------------------------------------------------------- ranges
// Blocks are laid out per batch element (gridDim.x = B * bpb): block j of
// element b owns a contiguous slice of that element's points, so a block
// histogram needs only K bins, whatever B is.  lo/hi are flat (b*N + i).
__device__ __forceinline__ void range_of(int64_t N, int bpb, int64_t& b, int64_t& lo,
                                         int64_t& hi) {
  b = blockIdx.x / bpb;
  const int j = blockIdx.x - (int)b * bpb;
  const int64_t per = (N + bpb - 1) / bpb;
  lo = b * N + (int64_t)j * per;
  const int64_t end = (int64_t)j * per + per < N ? (int64_t)j * per + per : N;
  hi = b * N + end;
  if (lo > hi) lo = hi;
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


// ----------------------------------------------------------------- hist
// Each block histograms its contiguous point range into its row of `table`
// (B*bpb rows of K int32).  K <= HIST_SMEM_KEYS: shared-memory bins, the whole
// row written out (zeros included); larger K: warp-aggregated atomics straight
// into the (pre-zeroed) global row.  Integer counts are order-independent.
// The blocks also clear, a grid-strided slice each, the f64 sums (unless the
// update accumulates) and the per-key arrival counters of k_segsum's ordered
// merge -- no separate memsets.
__global__ void __launch_bounds__(1024)
    k_hist(const int32_t* __restrict__ ids, int64_t N, int64_t K, int bpb, int32_t* __restrict__ table,
           double* __restrict__ zero_sums, int64_t zero_n, int32_t* __restrict__ arrive,
           int64_t arrive_n, int32_t* __restrict__ inval) {
  extern __shared__ int32_t sh[];
  __shared__ int32_t s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  {
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (zero_sums) {
      if ((reinterpret_cast<uintptr_t>(zero_sums) & 15) == 0) {  // 16-byte stores
        double2* z2 = reinterpret_cast<double2*>(zero_sums);
        for (int64_t i = t0; i < (zero_n >> 1); i += nt) z2[i] = make_double2(0.0, 0.0);
        if ((zero_n & 1) && t0 == 0) zero_sums[zero_n - 1] = 0.0;
      } else {
        for (int64_t i = t0; i < zero_n; i += nt) zero_sums[i] = 0.0;
      }
    }
    for (int64_t i = t0; i < arrive_n; i += nt) arrive[i] = 0;
  }
  const bool use_smem = K <= HIST_SMEM_KEYS;
  int64_t b, lo, hi;
  range_of(N, bpb, b, lo, hi);
  int32_t* trow = table + (int64_t)blockIdx.x * K;
  if (use_smem)
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) sh[k] = 0;
  __syncthreads();
  int bad = 0;
  for_each_id(ids, lo, hi, [&](int64_t, int32_t id) {
    if (id < 0 || id >= K) {  // not a cluster: left out of the sort (and the sums)
      ++bad;
      return;
    }
    if (use_smem) {
      atomicAdd(&sh[id], 1);
    } else {
      const unsigned peers = __match_any_sync(__activemask(), id);
      if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&trow[id], __popc(peers));
    }
  });
  for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&s_bad, bad);
  __syncthreads();
  if (use_smem)
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) trow[k] = sh[k];
  if (inval && threadIdx.x == 0) inval[blockIdx.x] = s_bad;
}

// ----------------------------------------------------------------- colscan
// Per key, over the bpb block rows of its batch element in block order:
// table[blk][k] <- sum of table[blk'][k] for blk' < blk (where block blk's
// points of key k start inside the key's run), and hist[b*K + k] <- the total.
// Block (32 keys) x (32 row groups): coalesced 128-byte row reads.
__global__ void __launch_bounds__(1024)
    k_colscan(int32_t* __restrict__ table, int64_t K, int bpb, int64_t ktiles,
              int32_t* __restrict__ hist) {
  __shared__ int32_t part[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t b = blockIdx.x / ktiles;
  const int64_t k = (blockIdx.x - b * ktiles) * 32 + tx;
  const int R = (bpb + 31) / 32;
  const int r0 = ty * R < bpb ? ty * R : bpb;
  const int r1 = r0 + R < bpb ? r0 + R : bpb;
  int32_t* col = table + (int64_t)b * bpb * K + k;
  int32_t s = 0;
  if (k < K)
    for (int r = r0; r < r1; ++r) s += col[(int64_t)r * K];
  part[ty][tx] = s;
  __syncthreads();
  int32_t pre = 0;
  for (int q = 0; q < ty; ++q) pre += part[q][tx];
  if (k < K) {
    for (int r = r0; r < r1; ++r) {
      const int32_t c = col[(int64_t)r * K];
      col[(int64_t)r * K] = pre;
      pre += c;
    }
    if (ty == 31) hist[b * K + k] = pre;
  }
}

// ----------------------------------------------------------------- scan
// One block of 1024 threads per batch element b.  The block first reduces the
// histogram of all earlier batch elements (its base offset; b*N when every id
// is valid), then walks its own K keys in tiles of 4096 (4 consecutive keys
// per thread, so K <= 4096 is one pass): block-wide exclusive scan per tile
// plus a running carry.  Also produces the int64 counts and the reference's
// synchronized_merges count.  off[B*K] = number of sorted (valid) points.
__global__ void __launch_bounds__(1024)
    k_scan(const int32_t* __restrict__ hist, int64_t B, int64_t N, int64_t K, int64_t chunk,
           int accumulate, int64_t* __restrict__ off, int64_t* __restrict__ counts,
           int64_t* __restrict__ merges) {
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
  const int64_t base_b = carry;  // start of this batch element's runs
  __syncthreads();
  unsigned long long mg = 0;
  const uint32_t ch = (uint32_t)chunk;
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
        if (counts) counts[k] = accumulate ? counts[k] + c[q] : c[q];
        if (c[q] > 0 && merges) {
          // reference merges: the run [s, e) of this key inside its batch element
          // meets floor((e-1)/chunk) - floor(s/chunk) + 1 update chunks
          // (all quantities < 2^31: 32-bit divisions)
          const uint32_t s0 = (uint32_t)(run - base_b), e = s0 + (uint32_t)c[q];
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
// Stable counting sort of the point indices by id.  Each block walks its range
// in sub-tiles of SD_S points; a sub-tile is sorted in shared memory by LSD
// radix passes of <= 8 bits: warp w owns SD_PW consecutive positions of the
// current order, counts digits per (digit, warp) (one counter update per
// distinct digit per warp step, warp-private, no atomics), a block scan in
// digit-major/warp-minor order gives every (digit, warp) its base, and a
// second walk in the same order places the elements -- stable by construction.
// The sorted sub-tile is written at off[key] + (block base of the key, from
// k_colscan, advanced by earlier sub-tiles) + rank in the key's run: the
// global order is the stable argsort of the ids (_kernels.py:118-132).
constexpr int SD_T = 1024;              // threads per block (one block per SM)
constexpr int SD_W = SD_T / 32;         // warps
constexpr int SD_S = 8192;              // points per sub-tile
constexpr int SD_PW = SD_S / SD_W;      // positions per warp
constexpr int SD_PT = SD_S / SD_T;      // positions per thread (blocked phases)
constexpr int SD_KSMEM = 4096;          // K up to this: the block's key bases live in smem
constexpr size_t SD_SMEM = (size_t)SD_S * 4 + 2 * (size_t)SD_S * 2 + 256 * SD_W * 4;
constexpr size_t SD_SMEM_BASES = SD_SMEM + (size_t)SD_KSMEM * 4;

// Exclusive block scan (SD_T threads) of one value per thread; *total = sum.
template <typename Op>
__device__ __forceinline__ int sd_block_scan(int v, int ident, int* wbuf, int* total, Op op) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = op(incl, u);
  }
  int excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = ident;
  if (lane == 31) wbuf[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < SD_W ? wbuf[lane] : ident;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x = op(x, u);
    }
    if (lane < SD_W) wbuf[lane] = x;  // inclusive over warps
  }
  __syncthreads();
  const int res = w ? op(wbuf[w - 1], excl) : excl;
  if (total) *total = wbuf[SD_W - 1];
  __syncthreads();
  return res;
}

// Lanes holding the same digit as this lane, among `valid`.  MATCH = 1 uses
// match.any; otherwise one ballot per digit bit (CUB's MatchAny).
template <bool MATCH>
__device__ __forceinline__ unsigned sd_peers(uint32_t dg, int nbits, bool valid) {
  if (MATCH) return __match_any_sync(0xffffffffu, valid ? dg : 0x10000u | (threadIdx.x & 31)) &
                    __ballot_sync(0xffffffffu, valid);
  unsigned m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i < nbits) {
      const bool bit = (dg >> i) & 1u;
      const unsigned bal = __ballot_sync(0xffffffffu, bit);
      m &= bit ? bal : ~bal;
    }
  }
  return m;
}

template <int NP, bool SBASE, bool MATCH>
__global__ void __launch_bounds__(SD_T, 1)
    k_scatter_stable(const int32_t* __restrict__ ids, int64_t N, int64_t K, int bpb, int last_bits,
                     int32_t* __restrict__ table, const int64_t* __restrict__ off,
                     int32_t* __restrict__ order) {
  extern __shared__ __align__(16) uint8_t sd_sm[];
  uint32_t* skey = reinterpret_cast<uint32_t*>(sd_sm);
  uint16_t* pa = reinterpret_cast<uint16_t*>(skey + SD_S);
  uint16_t* pb = pa + SD_S;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(pb + SD_S);
  int32_t* sbase = reinterpret_cast<int32_t*>(cnt + 256 * SD_W);  // SBASE: next position per key
  __shared__ int wbuf[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const auto add = [](int a, int b) { return a + b; };
  const auto mx = [](int a, int b) { return a > b ? a : b; };
  int64_t b, lo, hi;
  range_of(N, bpb, b, lo, hi);
  int32_t* trow = table + (int64_t)blockIdx.x * K;
  const int64_t* offb = off + b * K;
  if (SBASE)  // flat positions < 2^31 (B*N is): int32 bases, advanced in shared memory
    for (int k = t; k < K; k += SD_T) sbase[k] = (int32_t)(offb[k] + trow[k]);
  for (int64_t s0 = lo; s0 < hi; s0 += SD_S) {
    const int n = (int)(hi - s0 < SD_S ? hi - s0 : SD_S);
#pragma unroll 4
    for (int i = t; i < SD_S; i += SD_T) skey[i] = i < n ? (uint32_t)__ldg(ids + s0 + i) : 0xffffffffu;
    __syncthreads();
    int nv = n;
    uint16_t* src = pa;
    uint16_t* dst = pb;
#pragma unroll
    for (int pass = 0; pass < NP; ++pass) {
      const int shift = 8 * pass;
      const int nbits = pass == NP - 1 ? last_bits : 8;
      const uint32_t dmask = (1u << nbits) - 1u;
      const int E = (1 << nbits) * SD_W;  // (digit, warp) counters
      for (int i = t; i < E; i += SD_T) cnt[i] = 0;
      __syncthreads();
      // count walk (pass 0 visits the sub-tile in index order and drops ids
      // outside [0, K): they are not points of any cluster).  This lane's
      // digits and peer masks are kept for the scatter walk.
      uint32_t dge[SD_PW / 32];  // digit << 16 | local index, or ~0 for no element
      unsigned pes[SD_PW / 32];
#pragma unroll
      for (int st = 0; st < SD_PW / 32; ++st) {
        const int pos = w * SD_PW + st * 32 + lane;
        bool valid;
        uint32_t e, k;
        if (pass == 0) {
          e = (uint32_t)pos;
          k = skey[pos];
          valid = pos < n && k < (uint32_t)K;
        } else {
          valid = pos < nv;
          e = valid ? src[pos] : 0u;
          k = skey[e];
        }
        const uint32_t dg = (k >> shift) & dmask;
        const unsigned peers = sd_peers<MATCH>(dg, nbits, valid);
        dge[st] = valid ? (dg << 16 | e) : 0xffffffffu;
        pes[st] = peers;
      }
      // per-(digit, warp) counts: the lowest lane of each digit group adds the
      // group's size, one step after another (warp-private counters)
#pragma unroll
      for (int st = 0; st < SD_PW / 32; ++st) {
        if (dge[st] != 0xffffffffu && (pes[st] & lt) == 0) cnt[(dge[st] >> 16) * SD_W + w] += (uint32_t)__popc(pes[st]);
        __syncwarp();
      }
      __syncthreads();
      {  // exclusive scan of the counters, digit-major / warp-minor
        const int per = E >= SD_T ? E / SD_T : 1;
        const int i0 = t * per;
        uint32_t v[8];
        int sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[j] = (j < per && i0 + j < E) ? cnt[i0 + j] : 0u;
          sum += (int)v[j];
        }
        int tot;
        int ex = sd_block_scan(sum, 0, wbuf, &tot, add);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < per && i0 + j < E) {
            cnt[i0 + j] = (uint32_t)ex;
            ex += (int)v[j];
          }
        if (pass == 0) nv = tot;
      }
      __syncthreads();
      // scatter walk: same positions in the same order
#pragma unroll
      for (int st = 0; st < SD_PW / 32; ++st) {
        const bool ok = dge[st] != 0xffffffffu;
        const uint32_t dg = dge[st] >> 16;
        const unsigned peers = pes[st];
        uint32_t base = 0;
        if (ok) {
          base = cnt[dg * SD_W + w];
          dst[base + __popc(peers & lt)] = (uint16_t)(dge[st] & 0xffffu);
        }
        __syncwarp();
        if (ok && (peers & lt) == 0) cnt[dg * SD_W + w] = base + (uint32_t)__popc(peers);
        __syncwarp();
      }
      __syncthreads();
      uint16_t* tmp = src;
      src = dst;
      dst = tmp;
    }
    // src[0, nv): the sub-tile's local indices stably sorted by id.  Run starts,
    // blocked (thread t owns positions [SD_PT*t, SD_PT*t + SD_PT)), into dst.
    {
      const int p0 = SD_PT * t;
      uint32_t kp = (p0 > 0 && p0 - 1 < nv) ? skey[src[p0 - 1]] : 0xffffffffu;
      int rs[SD_PT];
      int m = -1;
#pragma unroll
      for (int j = 0; j < SD_PT; ++j) {
        const int p = p0 + j;
        if (p < nv) {
          const uint32_t k = skey[src[p]];
          if (k != kp || p == 0) m = p;
          kp = k;
        }
        rs[j] = m;
      }
      const int carry = sd_block_scan(m, -1, wbuf, nullptr, mx);
#pragma unroll
      for (int j = 0; j < SD_PT; ++j)
        if (p0 + j < nv) dst[p0 + j] = (uint16_t)(rs[j] >= 0 ? rs[j] : carry);
    }
    __syncthreads();
    // write the order (strided: a warp stores 32 consecutive positions); every
    // base is fetched before the first store, then each run's end advances the
    // key's base for the next sub-tile
    int32_t gp[SD_PT];  // flat positions: B*N < 2^31
    uint32_t kk[SD_PT];
    bool endr[SD_PT];
#pragma unroll
    for (int j = 0; j < SD_PT; ++j) {
      const int p = j * SD_T + t;
      kk[j] = 0xffffffffu;
      endr[j] = false;
      if (p < nv) {
        const uint32_t k = skey[src[p]];
        const int r = p - (int)dst[p];
        kk[j] = k;
        gp[j] = (int32_t)(SBASE ? sbase[k] : offb[k] + __ldcg(trow + k)) + r;
        endr[j] = p + 1 == nv || (int)dst[p + 1] == p + 1;
      }
    }
#pragma unroll
    for (int j = 0; j < SD_PT; ++j)
      if (kk[j] != 0xffffffffu) order[gp[j]] = (int32_t)(s0 + src[j * SD_T + t]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < SD_PT; ++j)
      if (endr[j]) {
        if (SBASE)
          sbase[kk[j]] = (int32_t)(gp[j] + 1);
        else
          __stcg(trow + kk[j], (int32_t)((int64_t)gp[j] + 1 - offb[kk[j]]));
      }
    __syncthreads();
  }
}

// Stable scatter for K <= SW_KMAX: warp-granular tables instead of a block
// sort.  Block = W warps; warp w owns a contiguous part of the block's range.
//   1. each warp counts its part into its own row of a (W, K) u16 table
//      (shared atomics: counts are order-independent);
//   2. per key, an exclusive prefix over the W rows (warp order = index
//      order), plus the key's global base off[key] + (block base, k_colscan);
//   3. each warp walks its part in index order, 32 points a step; every lane
//      takes its rank from a returning shared atomic on its warp's count.
// No match.any: its cost grows with the number of distinct values in the warp
// (scripts/probe_match.cu: ~2000 cycles per warp instruction at 32 distinct
// ids with 32 warps per SM, against ~65 for a conflicting shared atomic).
// The ids of SW_U steps are loaded together.  The u16 table needs block
// ranges < 2^16 points (update_bpb).
constexpr int SW_KMAX = 16384;            // W * (K + 2) * 2 bytes <= 64 KB, + K * 8 bytes of bases
constexpr int SW_TABLE_BYTES = 65536;
// Programmatic dependent launch (default; FK_PDL=0 turns it off for A/B): the
// scatter and the segsum release their dependents as soon as every CTA of
// theirs is resident, so the segsum / normalize CTAs are placed while the previous kernel drains; a
// dependent waits for its predecessor's completion (and memory) before any
// access.  Both instructions are no-ops for an ordinary launch.  Same-box A/B
// (profiles/r02_ab_pdl.txt): config-4 update 57.1-57.6 -> 54.4-54.8 us and
// the eagerly launched pipelined loop 3-5 us faster at configs 2/4; inside a
// CUDA graph the inter-kernel gaps are already hidden (no change).
FK_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
FK_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
FK_DEV void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}
static bool pdl_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FK_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
template <typename... KArgs, typename... Args>
static void launch_maybe_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem,
                             cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...);
}

constexpr int SW_U = 8;                   // 16-byte id vectors in flight per lane (counting)
constexpr int SW_U3 = 16;                 // id loads in flight per lane (ranking)
constexpr int SW_COLS_BPB = 16;           // up to this many blocks per batch element: no k_colscan

// Exclusive scan, in place, of n int32 values in shared memory by the whole
// block (T threads, contiguous chunks per thread); returns the total.
template <int T>
__device__ int sw_block_scan(int32_t* v, int n, int32_t* wsum) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  constexpr int NW = T / 32;
  const int per = (n + T - 1) / T;
  const int i0 = t * per < n ? t * per : n;
  const int i1 = i0 + per < n ? i0 + per : n;
  int sum = 0;
  for (int i = i0; i < i1; ++i) sum += v[i];
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < NW ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += u;
    }
    if (lane < NW) wsum[lane] = x;
  }
  __syncthreads();
  int run = incl - sum + (w ? wsum[w - 1] : 0);
  const int total = wsum[NW - 1];
  for (int i = i0; i < i1; ++i) {
    const int c = v[i];
    v[i] = run;
    run += c;
  }
  __syncthreads();
  return total;
}

// COLS: the block also does the column prefix over its batch element's bpb
// block rows (small bpb; otherwise k_colscan did it and wrote the totals to
// `hist`).  Every block then derives the key offsets of its batch element
// itself (exclusive scan of the totals + the batch element's base, b*N minus
// the ids outside [0, K) of earlier elements); block 0 of each batch element
// also publishes off[], the int64 counts and the reference merge count -- no
// separate scan kernel.
template <int W, bool COLS>
__global__ void __launch_bounds__(W * 32)
    k_scatter_warp(const int32_t* __restrict__ ids, int64_t N, int64_t K, int bpb,
                   const int32_t* __restrict__ table, const int32_t* __restrict__ hist,
                   const int32_t* __restrict__ inval, int64_t B, int64_t chunk, int accumulate,
                   int64_t* __restrict__ off, int64_t* __restrict__ counts, int64_t* __restrict__ merges,
                   int32_t* __restrict__ order, int rank_sort, double* __restrict__ zero_sums,
                   int64_t zero_n, int32_t* __restrict__ zero_arrive, int64_t arrive_n) {
  extern __shared__ __align__(16) uint8_t sw_sm[];
  pdl_trigger();
  // block histograms folded into the assign (no k_hist): this pass clears the
  // f64 sums and k_segsum's arrival counters instead
  if (zero_sums || zero_arrive) {
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (zero_sums) {
      if ((reinterpret_cast<uintptr_t>(zero_sums) & 15) == 0) {
        double2* z2 = reinterpret_cast<double2*>(zero_sums);
        for (int64_t i = t0; i < (zero_n >> 1); i += nt) z2[i] = make_double2(0.0, 0.0);
        if ((zero_n & 1) && t0 == 0) zero_sums[zero_n - 1] = 0.0;
      } else {
        for (int64_t i = t0; i < zero_n; i += nt) zero_sums[i] = 0.0;
      }
    }
    for (int64_t i = t0; i < arrive_n; i += nt) zero_arrive[i] = 0;
  }
  // rows padded to K + 2 entries: the W rows of one key fall in different banks
  const int KS = (int)K + 2;
  uint16_t* tab = reinterpret_cast<uint16_t*>(sw_sm);                           // W * KS
  int32_t* kbase = reinterpret_cast<int32_t*>(sw_sm + ((W * KS * 2 + 15) & ~15));  // K
  // the key prefix lives in the table's space when it fits (the table is
  // cleared only after the prefix is folded into kbase)
  const bool alias = (int64_t)W * KS * 2 >= K * 4;
  int32_t* kpre = alias ? reinterpret_cast<int32_t*>(sw_sm) : kbase + K;         // K
  uint32_t* tab32 = reinterpret_cast<uint32_t*>(sw_sm);
  __shared__ int32_t wsum[32];
  __shared__ unsigned long long s_bad, s_mg;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t Ku = (uint32_t)K;
  int64_t b, lo, hi;
  range_of(N, bpb, b, lo, hi);
  const int j = (int)(blockIdx.x - b * bpb);
  const int32_t* trow = table + (int64_t)blockIdx.x * K;
  if (t == 0) {
    s_bad = 0;
    s_mg = 0;
  }
  // block base inside each key's run (kbase) and the key totals (kpre)
#pragma unroll 4
  for (int k = t; k < K; k += W * 32) {
    if (COLS) {
      const int32_t* col = table + (int64_t)b * bpb * K + k;
      int32_t run = 0, tot = 0;
      for (int r = 0; r < bpb; ++r) {
        const int32_t c = col[(int64_t)r * K];
        run += r < j ? c : 0;
        tot += c;
      }
      kbase[k] = run;
      kpre[k] = tot;
    } else {
      kbase[k] = trow[k];
      kpre[k] = hist[b * K + k];
    }
  }
  {  // batch base: b*N minus the invalid ids of the earlier batch elements
    unsigned long long bad = 0;
    for (int64_t i = t; i < b * bpb; i += W * 32) bad += (unsigned long long)inval[i];
    for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    __syncthreads();
    if (lane == 0 && bad) atomicAdd(&s_bad, bad);
  }
  // key offsets relative to the batch element: exclusive prefix of the totals
  const int32_t total = sw_block_scan<W * 32>(kpre, (int)K, wsum);
  const int64_t base_b = b * N - (int64_t)s_bad;
  if (j == 0) {  // publish off / counts / merges for this batch element
    unsigned long long mg = 0;
    const uint32_t ch = (uint32_t)chunk;
    for (int k = t; k < K; k += W * 32) {
      const int32_t s0 = kpre[k];
      const int32_t c = (k + 1 < K ? kpre[k + 1] : total) - s0;
      off[b * K + k] = base_b + s0;
      if (counts) counts[b * K + k] = accumulate ? counts[b * K + k] + c : c;
      if (c > 0) mg += (unsigned long long)(((uint32_t)(s0 + c) - 1) / ch - (uint32_t)s0 / ch + 1);
    }
    if (b == B - 1 && t == 0) off[B * K] = base_b + total;
    for (int o = 16; o; o >>= 1) mg += __shfl_xor_sync(0xffffffffu, mg, o);
    if (lane == 0 && mg) atomicAdd(&s_mg, mg);
  }
  for (int k = t; k < K; k += W * 32) kbase[k] += (int32_t)(base_b + kpre[k]);  // flat < 2^31
  __syncthreads();  // kpre consumed: the table space is free
  for (int i = t; i < W * KS / 2; i += W * 32) tab32[i] = 0u;
  // this warp's part [a, e) of the block range
  const int n = (int)(hi - lo);
  const int a = (int)((int64_t)n * w / W), e = (int)((int64_t)n * (w + 1) / W);
  const int32_t* idw = ids + lo;
  __syncthreads();
  if (j == 0 && merges && t == 0 && s_mg) atomicAdd((unsigned long long*)merges, s_mg);
  // 1. per-warp counts (fire-and-forget shared atomics on packed u16 pairs);
  //    order-free, so the ids come in as 16-byte vectors (SW_U of them in flight)
  {
    auto count = [&](uint32_t id) {
      if (id < Ku) {
        const uint32_t f = (uint32_t)(w * KS) + id;
        atomicAdd(tab32 + (f >> 1), 1u << (16 * (f & 1)));
      }
    };
    // scalar head up to a 16-byte boundary of the ADDRESS (ids may be a slice
    // at any int32 offset, e.g. one streamed chunk)
    const uintptr_t ga = reinterpret_cast<uintptr_t>(idw + a);
    int h = (int)(((16 - (ga & 15)) & 15) >> 2);
    if (h > e - a) h = e - a;
    if (lane < h) count((uint32_t)__ldg(idw + a + lane));
    const int nv = (e - a - h) >> 2;
    const int4* v4 = reinterpret_cast<const int4*>(idw + a + h);
    for (int q0 = 0; q0 < nv; q0 += 32 * SW_U) {
      int4 v[SW_U];
#pragma unroll
      for (int u = 0; u < SW_U; ++u) {
        const int q = q0 + u * 32 + lane;
        v[u] = q < nv ? __ldg(v4 + q) : make_int4(-1, -1, -1, -1);
      }
#pragma unroll
      for (int u = 0; u < SW_U; ++u) {
        count((uint32_t)v[u].x);
        count((uint32_t)v[u].y);
        count((uint32_t)v[u].z);
        count((uint32_t)v[u].w);
      }
    }
    const int t0 = a + h + 4 * nv;
    if (lane < e - t0) count((uint32_t)__ldg(idw + t0 + lane));
  }
  __syncthreads();
  // 2. exclusive prefix over the W warp rows of each key: segmented warp scans
  //    of width W (32/W keys per warp instruction)
  {
    constexpr int KPW = 32 / W;  // keys per warp pass
    const int q = lane % W, ks = lane / W;
    for (int k0 = w * KPW; k0 < K; k0 += W * KPW) {
      const int k = k0 + ks;
      const uint32_t c = k < K ? tab[q * KS + k] : 0u;
      uint32_t v = c;
#pragma unroll
      for (int o = 1; o < W; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o, W);
        if (q >= o) v += u;
      }
      if (k < K) tab[q * KS + k] = (uint16_t)(v - c);
    }
  }
  __syncthreads();
  // 3. ranks in index order.  FK_SCATTER_RANK=sort: 32 points a step, the
  //    step's ids are sorted across the warp by (id, lane) with a shuffle
  //    bitonic network;
  //    the lane holding a sorted entry reads its id's running count from the
  //    warp's row, adds its position inside the id's run (ballot of run
  //    starts) and writes the point index; the last lane of each run stores
  //    the new count (one writer per id).  (id, lane) keys are unique, so the
  //    ranks are the stable ones (numpy's stable argsort,
  //    tests/test_gpu_kernels.py), with no returning atomics on the critical
  //    path -- but more instructions: slower (A/B record).  Default: every
  //    lane bumps its counter with a returning shared atomic (lanes of one
  //    instruction on one counter are served in lane order).  The ids are
  //    re-read (L2-resident).
  if (rank_sort) {
    for (int p0 = a; p0 < e; p0 += 32) {
      const int p = p0 + lane;
      const uint32_t id = p < e ? (uint32_t)__ldg(idw + p) : 0xffffffffu;
      uint32_t key = id < Ku ? ((id << 5) | (uint32_t)lane) : 0xffffffffu;
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, key, j);
          const bool up = (lane & k) == 0;       // ascending block
          const bool lower = (lane & j) == 0;    // this lane keeps the smaller key
          key = (lower == up) ? min(key, o) : max(key, o);
        }
      }
      const bool valid = key != 0xffffffffu;
      const uint32_t sid = key >> 5;
      const uint32_t prev = __shfl_up_sync(0xffffffffu, sid, 1);
      const uint32_t next = __shfl_down_sync(0xffffffffu, sid, 1);
      const bool first = lane == 0 || prev != sid;
      const bool last = lane == 31 || next != sid;
      const unsigned starts = __ballot_sync(0xffffffffu, first);
      const int run0 = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));
      if (valid) {
        uint16_t* cnt = tab + w * KS + sid;
        const uint32_t r = (uint32_t)*cnt + (uint32_t)(lane - run0);
        order[kbase[sid] + (int32_t)r] = (int32_t)(lo + p0 + (int)(key & 31u));
        if (last) *cnt = (uint16_t)(r + 1);
      }
      __syncwarp();
    }
    return;
  }
  for (int p0 = a; p0 < e; p0 += 32 * SW_U3) {
    uint32_t id[SW_U3];
#pragma unroll
    for (int u = 0; u < SW_U3; ++u) {
      const int p = p0 + u * 32 + lane;
      id[u] = p < e ? (uint32_t)__ldg(idw + p) : 0xffffffffu;
    }
#pragma unroll
    for (int u = 0; u < SW_U3; ++u)
      if (id[u] < Ku) {
        const uint32_t f = (uint32_t)(w * KS) + id[u];
        const uint32_t sh = 16 * (f & 1);
        const uint32_t r = (atomicAdd(tab32 + (f >> 1), 1u << sh) >> sh) & 0xffffu;
        order[kbase[id[u]] + (int32_t)r] = (int32_t)(lo + p0 + u * 32 + lane);
      }
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

// One merge per (slice, segment).  A segment inside the slice is stored
// directly.  A segment spanning slices [w0, w1] leaves its partial in slot
// part[w][s] (s = 0 when the segment contains the slice's first position, else
// 1), and the last slice to arrive (per-key counter) adds the partials in
// slice order w0..w1 -- the reference's ascending merge order, whichever
// warp finishes last.  `acc_j(j)` gives this lane's partial of column j, for
// the columns `for_cols` visits.
struct SegMerge {
  double* part;     // [slices][2][d] f64 partials of segments spanning slices
  int32_t* arrive;  // [B*K] arrival counters (zeroed by k_hist)
  int64_t L, d;
  int32_t* zero_i32;  // histogram folded into the assign: the block table + invalid
  int64_t zero_n;     // counts, cleared here for the next assign (nullptr: none)
};

// k_segsum* run after the scatter, the last reader of the block table
FK_DEV void seg_zero_table(const SegMerge& m) {
  if (!m.zero_i32) return;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(m.zero_i32) & 15) == 0) {
    int4* z4 = reinterpret_cast<int4*>(m.zero_i32);
    for (int64_t i = t0; i < (m.zero_n >> 2); i += nt) z4[i] = make_int4(0, 0, 0, 0);
    for (int64_t i = (m.zero_n & ~int64_t(3)) + t0; i < m.zero_n; i += nt) m.zero_i32[i] = 0;
  } else {
    for (int64_t i = t0; i < m.zero_n; i += nt) m.zero_i32[i] = 0;
  }
}

FK_DEV void seg_flush_boundary(const SegMerge& m, int64_t wg, int64_t p0, int64_t key, int64_t seg_lo,
                               int64_t seg_end, double* __restrict__ dst) {
  // the caller has written its partial into part[wg][slot] and fenced
  const int lane = threadIdx.x & 31;
  __syncwarp();
  int last = 0;
  const int64_t w0 = seg_lo / m.L, w1 = (seg_end - 1) / m.L;
  if (lane == 0) {
    const int old = atomicAdd(m.arrive + key, 1);
    last = old == (int)(w1 - w0);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  const int64_t s0 = (seg_lo == w0 * m.L) ? 0 : 1;
  for (int64_t j = lane; j < m.d; j += 32) {
    double tot = __ldcg(m.part + (w0 * 2 + s0) * m.d + j);
    for (int64_t w = w0 + 1; w <= w1; ++w) tot += __ldcg(m.part + (w * 2) * m.d + j);
    dst[j] += tot;
  }
  (void)p0;
  (void)wg;
}

// LPR lanes cover one row with VPL 16-byte vectors each; RPW = 32/LPR rows per
// warp step; U steps are issued back to back to keep bytes in flight.
template <typename T, typename A, int LPR, int VPL, int U>
__global__ void __launch_bounds__(256)
    k_segsum(const T* __restrict__ X, const int32_t* __restrict__ order,
             const int64_t* __restrict__ off, int64_t BK, int64_t L, int64_t d,
             double* __restrict__ sums, const int32_t* __restrict__ ids, int64_t N, int64_t K,
             SegMerge mg) {
  pdl_enter();
  seg_zero_table(mg);
  constexpr int E = VecCvt<T>::E;
  constexpr int RPW = 32 / LPR;
  constexpr int NA = VPL * E;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, sl = lane % LPR;
  const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t P = off[BK];  // sorted (valid) points
  const int64_t p0 = wg * L;
  if (p0 >= P) return;
  const int64_t p1 = (p0 + L < P) ? p0 + L : P;
  // segment containing p0 (largest key with off[key] <= p0 < off[key+1]) is
  // the key of the point sorted to p0: two dependent loads instead of a
  // log2(BK)-step binary search over off[]
  const int32_t pt = order[p0];
  const int64_t pb = pt / N;
  int64_t key = pb * K + ids[pt];
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
    // flush this segment's partial (one merge per segment; fixed shuffle tree)
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
      for (int e = 0; e < NA; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    double* dst = sums + key * d;
    if (seg_lo >= p0 && seg_end <= p1) {  // owned: the only writer of this key
      if (sub == 0) {
#pragma unroll
        for (int q = 0; q < VPL; ++q)
#pragma unroll
          for (int e = 0; e < E; ++e) dst[(int64_t)(q * LPR + sl) * E + e] += (double)acc[q * E + e];
      }
    } else {
      double* pp = mg.part + (wg * 2 + (seg_lo <= p0 ? 0 : 1)) * d;
      if (sub == 0) {
#pragma unroll
        for (int q = 0; q < VPL; ++q)
#pragma unroll
          for (int e = 0; e < E; ++e) pp[(int64_t)(q * LPR + sl) * E + e] = (double)acc[q * E + e];
        __threadfence();
      }
      seg_flush_boundary(mg, wg, p0, key, seg_lo, seg_end, dst);
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

// Segment-chained variant (default).  Same slices, same per-segment groups
// and addition order as k_segsum, but the transitions between segments cost
// no dependent loads: the segment ends come from a 32-key window of off[]
// held one per lane (one refill per 32 keys), the indices of the NEXT group
// -- this segment's next group or the next segment's first -- are prefetched
// while the current group's rows are in flight (the old tail group and the
// next segment's first group each waited for their indices, then for their
// rows), and an owned segment of a non-accumulating update is stored without
// reading the cleared sums back.  Positions are 32-bit (sorted points <
// 2^31, as the scatter's flat offsets).
template <typename T, typename A, int LPR, int VPL, int U>
__global__ void __launch_bounds__(256, sizeof(A) == 8 ? 3 : 4)
    k_segsum2(const T* __restrict__ X, const int32_t* __restrict__ order,
              const int64_t* __restrict__ off, int64_t BK, int64_t L, int64_t d,
              double* __restrict__ sums, const int32_t* __restrict__ ids, int64_t N, int64_t K,
              SegMerge mg, int accumulate) {
  pdl_enter();
  seg_zero_table(mg);
  constexpr int E = VecCvt<T>::E;
  constexpr int RPW = 32 / LPR;
  constexpr int NA = VPL * E;
  constexpr int G = RPW * U;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, sl = lane % LPR;
  const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int P = (int)off[BK];
  if (wg * L >= P) return;
  const int p0 = (int)(wg * L);
  const int p1 = p0 + L < P ? p0 + (int)L : P;
  const int32_t pt = order[p0];
  const int pb = pt / (int)N;
  int key = pb * (int)K + ids[pt];
  int wb = key;  // window: lane i holds off[wb + 1 + i]
  int win = wb + 1 + lane <= BK ? (int)off[wb + 1 + lane] : INT_MAX;
  int seg_lo = (int)off[key];
  int seg_end = __shfl_sync(0xffffffffu, win, 0);
  auto end_of = [&](int k) -> int {
    if (k - wb >= 32) {
      wb = k;
      win = wb + 1 + lane <= BK ? (int)off[wb + 1 + lane] : INT_MAX;
    }
    return __shfl_sync(0xffffffffu, win, k - wb);
  };
  A acc[NA];
#pragma unroll
  for (int e = 0; e < NA; ++e) acc[e] = (A)0;
  int p = p0;
  int lim = seg_end < p1 ? seg_end : p1;
  int32_t ri[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int r = p + u * RPW + sub;
    ri[u] = r < lim ? __ldg(order + r) : -1;
  }
  while (true) {
    uint4 v[U][VPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const T* rp = X + (int64_t)(ri[u] < 0 ? 0 : ri[u]) * d;
#pragma unroll
      for (int q = 0; q < VPL; ++q)
        v[u][q] = ri[u] >= 0 ? ldg_stream(rp + (q * LPR + sl) * E) : make_uint4(0u, 0u, 0u, 0u);
    }
    const bool done = p + G >= lim;  // this group ends the segment's part of the slice
    int nkey = key, nlo = seg_lo, nend = seg_end, nlim = lim, np = p + G;
    if (done && lim < p1) {  // the next non-empty segment starts at lim
      nlo = lim;
      do nend = end_of(++nkey);
      while (nend <= nlo);
      nlim = nend < p1 ? nend : p1;
      np = nlo;
    }
    if (!done || lim < p1) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = np + u * RPW + sub;
        ri[u] = r < nlim ? __ldg(order + r) : -1;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < VPL; ++q) VecCvt<T>::add(acc + q * E, v[u][q]);
    if (done) {
      // flush the segment's partial (one merge per segment; fixed shuffle tree)
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
        for (int e = 0; e < NA; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
      double* dst = sums + (int64_t)key * d;
      if (seg_lo >= p0 && seg_end <= p1) {  // owned: the only writer of this key
        if (sub == 0) {
#pragma unroll
          for (int q = 0; q < VPL; ++q)
#pragma unroll
            for (int e = 0; e < E; ++e) {
              double* o = dst + (int64_t)(q * LPR + sl) * E + e;
              *o = __dadd_rn(accumulate ? *o : 0.0, (double)acc[q * E + e]);
            }
        }
      } else {
        double* pp = mg.part + (wg * 2 + (seg_lo <= p0 ? 0 : 1)) * d;
        if (sub == 0) {
#pragma unroll
          for (int q = 0; q < VPL; ++q)
#pragma unroll
            for (int e = 0; e < E; ++e) pp[(int64_t)(q * LPR + sl) * E + e] = (double)acc[q * E + e];
          __threadfence();
        }
        seg_flush_boundary(mg, wg, p0, key, seg_lo, seg_end, dst);
      }
#pragma unroll
      for (int e = 0; e < NA; ++e) acc[e] = (A)0;
      if (lim >= p1) break;
      key = nkey;
      seg_lo = nlo;
      seg_end = nend;
      lim = nlim;
    }
    p = np;
  }
}

// Any row width: one warp per slice, lanes stride over the features.
template <typename T>
__global__ void k_segsum_generic(const T* __restrict__ X, const int32_t* __restrict__ order,
                                 const int64_t* __restrict__ off, int64_t BK, int64_t L, int64_t d,
                                 double* __restrict__ sums, SegMerge mg) {
  seg_zero_table(mg);
  const int lane = threadIdx.x & 31;
  const int64_t wg = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t P = off[BK];
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
    double* dst = sums + key * d;
    double* pp = mg.part + (wg * 2 + (seg_lo <= p0 ? 0 : 1)) * d;
    for (int64_t j0 = 0; j0 < d; j0 += 32) {
      const int64_t j = j0 + lane;
      double acc = 0.0;
      if (j < d) {
        for (int64_t r = p; r < lim; ++r) acc += as_f64(X[(int64_t)order[r] * d + j]);
        if (owned) dst[j] += acc;
        else pp[j] = acc;
      }
    }
    if (!owned) {
      __threadfence();
      seg_flush_boundary(mg, wg, p0, key, seg_lo, seg_end, dst);
    }
    p = lim;
    if (p < p1) {
      ++key;
      while (off[key + 1] <= p) ++key;
    }
  }
}

// Blocks per batch element for the histogram / scatter passes: ~2 waves in
// total, each block owning >= 8192 points (one stable-sort sub-tile) so the
// per-block K-bin table, its column scan and the sort amortize.  For K beyond
// the shared bins the block rows live in global memory: keep them at most
// ~2 bytes per point.
static int64_t update_bpb(int64_t B, int64_t N, int64_t K, int num_sms) {
  // ~2 blocks per SM (4 per SM measured no faster at config 3: the larger
  // tables cost k_hist and k_colscan what the scatter gained)
  static int bps = -1;  // FK_UPDATE_BPS: histogram/scatter blocks per SM (A/B)
  if (bps < 0) {
    const char* e = getenv("FK_UPDATE_BPS");
    bps = e ? atoi(e) : 2;
    if (bps < 1 || bps > 16) bps = 2;
  }
  int64_t bpb = ((int64_t)num_sms * bps + B - 1) / B;
  static int minpts = -1;  // FK_UPDATE_MINPTS: fewest points per block for the warp scatter (A/B)
  if (minpts < 0) {
    const char* e = getenv("FK_UPDATE_MINPTS");
    minpts = e ? atoi(e) : SD_S;
    if (minpts < 256 || minpts > SD_S) minpts = SD_S;
  }
  const int64_t per_min = K <= SW_KMAX ? minpts : SD_S;
  const int64_t max_bpb = (N + per_min - 1) / per_min;
  if (bpb > max_bpb) bpb = max_bpb;
  if (K > HIST_SMEM_KEYS) {
    const int64_t cap = N / (2 * K);
    if (bpb > cap) bpb = cap;
  }
  const int64_t min_bpb = (N + 65534) / 65535;  // k_scatter_warp's u16 tables: ranges < 2^16
  if (bpb < min_bpb) bpb = min_bpb;
  return bpb < 1 ? 1 : bpb;
}
constexpr int kMaxSms = 256;  // workspace bound for any sm_100 part
constexpr int64_t kF64MaxSpans = 1024;  // f64 pieces path: update_chunk >= N / 1024
constexpr int kSegWarpsPerSm = 32;

// Slice length of k_segsum: 32 warp slices per SM (same-box A/B,
// profiles/r01_ab_segsum.txt: 64 -> 32 took config 2 from 67.8 to 64.1 us
// and config 4 from 52 to 49.5 us, config 3 unchanged; 16 starves config 3
// of bytes in flight), at least 64 points each.
static bool segsum_seq() {
  static int seq_env = -1;  // FK_SEGSUM_SEQ=1: the per-segment k_segsum (A/B)
  if (seq_env < 0) {
    const char* e = getenv("FK_SEGSUM_SEQ");
    seq_env = (e && e[0] == '1') ? 1 : 0;
  }
  return seq_env == 1;
}
// k_segsum2 for short segments only (<= 256 points per key on average:
// config 4, 64 per key: update 59.0 -> 56.2 us); with long segments the
// per-segment k_segsum's 8 row steps beat its 6 (config 2: 80.5 vs 86 us,
// config 3: 464 vs 473 us; profiles/r02_ab_segsum2.txt)
static bool segsum_chained(int64_t P, int64_t BK) { return !segsum_seq() && P <= 256 * BK; }
// k_segsum2 with f64 accumulators (f32 / f64 data) holds 3 blocks per SM
// (80 registers), the 2-byte types 4: one slice per resident warp
static int64_t segsum_slice(int64_t P, int64_t BK, int num_sms, int dt) {
  static int wps = -1;  // FK_SEGSUM_WPS: warp slices per SM (A/B)
  if (wps < 0) {
    const char* e = getenv("FK_SEGSUM_WPS");
    wps = e ? atoi(e) : 0;
    if (wps < 1 || wps > 64) wps = 0;
  }
  const int w = wps ? wps : (segsum_chained(P, BK) && (dt == DT_F32 || dt == DT_F64)) ? 24 : kSegWarpsPerSm;
  const int64_t want = (int64_t)num_sms * w;
  int64_t L = (P + want - 1) / want;
  return L < 64 ? 64 : L;
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


// Workspace: table (B*bpb*K) | hist (B*K) | off (B*K+1) | order (B*N) |
// arrive (B*K) | segment partials (slices * 2 * d f64).
struct UpdateWs {
  int32_t* table;
  int32_t* hist;
  int64_t* off;
  int32_t* order;
  int32_t* arrive;
  double* part;
  int32_t* inval;
  int64_t zero_n;  // int32 words from table through inval
};

static size_t update_ws_layout(int dt, int64_t B, int64_t N, int64_t K, int64_t d, int num_sms, void* base,
                               UpdateWs* ws) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const int64_t BK = B * K, P = B * N;
  const int64_t bpb = update_bpb(B, N, K, num_sms);
  const int64_t slices = (P + segsum_slice(P, BK, num_sms, dt) - 1) / segsum_slice(P, BK, num_sms, dt);
  // segment partials: per-slice boundary partials, or the f64 path's pieces
  // (B * (K + kF64MaxSpans) rows of d)
  const int64_t spans = N < kF64MaxSpans ? N : kF64MaxSpans;
  const size_t part = std::max((size_t)slices * 2 * d * 8,
                               dt == DT_F64 ? (size_t)(B * (K + spans)) * d * 8 : (size_t)0);
  // table and inval adjacent: one range to clear when the assign builds them
  const size_t sz[7] = {al((size_t)B * bpb * K * 4), al((size_t)B * bpb * 4), al((size_t)BK * 4),
                        al((size_t)(BK + 1) * 8),    al((size_t)P * 4),       al((size_t)BK * 4),
                        al(part)};
  size_t total = 0;
  uint8_t* p = static_cast<uint8_t*>(base);
  void* ptrs[7];
  for (int i = 0; i < 7; ++i) {
    ptrs[i] = p ? p + total : nullptr;
    total += sz[i];
  }
  if (ws) {
    ws->table = (int32_t*)ptrs[0];
    ws->inval = (int32_t*)ptrs[1];
    ws->hist = (int32_t*)ptrs[2];
    ws->off = (int64_t*)ptrs[3];
    ws->order = (int32_t*)ptrs[4];
    ws->arrive = (int32_t*)ptrs[5];
    ws->part = (double*)ptrs[6];
    ws->zero_n = (int64_t)((sz[0] + (size_t)B * bpb * 4) / 4);
  }
  return total;
}

size_t update_workspace_bytes(int dt, int64_t B, int64_t N, int64_t K, int64_t d) {
  // blocks and slices grow with the SM count: size for the largest sm_100 part
  return update_ws_layout(dt, B, N, K, d, kMaxSms, nullptr, nullptr);
}

// ------------------------------------------------------- serial f64 segsum
// f64 data (the reference's default precision): f64 addition of f64 addends
// is not associative, so the sums must follow the reference's order exactly
// (sort_inverse.py:106-149, _kernels.py:135-171): per batch element the stable
// sorted order is cut into spans of `chunk` positions; each (span, key) run is
// summed serially from 0.0 in sorted order (segment_stats), and the runs are
// merged into the key's sum in ascending span order, again from 0.0
// (merge_segments).  A streamed chunk's result is added to the running sums
// (PartialStats.combine, pipeline.py:250-257) when `accumulate`.
// Two kernels, so that a key's run is cut at the span boundaries into pieces
// that are summed in parallel (the serial critical path is one piece, not one
// cluster): k_seg_pieces, one warp per (key, piece, 32 features), sums its
// piece serially from 0.0 in sorted order into slot key + span (a key's
// pieces occupy consecutive spans, so slots never collide); k_seg_fold, one
// thread per (key, feature), folds the key's pieces in span order from 0.0.
// Rows are gathered U ahead of the dependent adds.
template <int U>
__global__ void __launch_bounds__(256)
    k_seg_pieces(const double* __restrict__ X, const int32_t* __restrict__ order,
                 const int64_t* __restrict__ off, int64_t BK, int64_t K, int d, int fgs,
                 int64_t chunk, int64_t ns, int jw, double* __restrict__ part) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= BK * jw * fgs) return;
  const int64_t key = warp / ((int64_t)jw * fgs);
  const int64_t rem = warp - key * jw * fgs;
  const int j0 = (int)(rem / fgs);
  const int f = (int)(rem - (int64_t)j0 * fgs) * 32 + lane;
  const bool act = f < d;
  const int64_t b = key / K;
  const int64_t s = off[key], e = off[key + 1], base = off[b * K];
  if (e <= s) return;
  const int64_t m0 = (s - base) / chunk, m1 = (e - 1 - base) / chunk;  // spans of the key's run
  for (int64_t m = m0 + j0; m <= m1; m += jw) {
    const int64_t p0 = s > base + m * chunk ? s : base + m * chunk;
    const int64_t p1 = e < base + (m + 1) * chunk ? e : base + (m + 1) * chunk;
    double acc = 0.0;
    // the sorted-order indices of the next U rows are fetched while this
    // batch's rows are in flight
    int32_t ri[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ri[u] = p0 + u < p1 ? __ldg(order + p0 + u) : 0;
    for (int64_t q0 = p0; q0 < p1; q0 += U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = (act && q0 + u < p1) ? __ldg(X + (int64_t)ri[u] * d + f) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) ri[u] = q0 + U + u < p1 ? __ldg(order + q0 + U + u) : 0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u < p1) acc = __dadd_rn(acc, v[u]);
    }
    if (act) part[((key - b * K) + b * (K + ns) + m) * d + f] = acc;
  }
}

__global__ void __launch_bounds__(256)
    k_seg_fold(const int64_t* __restrict__ off, int64_t BK, int64_t K, int d, int64_t chunk,
               int64_t ns, const double* __restrict__ part, double* __restrict__ sums,
               int accumulate) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= BK * d) return;
  const int64_t key = i / d;
  const int f = (int)(i - key * d);
  const int64_t b = key / K;
  const int64_t s = off[key], e = off[key + 1], base = off[b * K];
  double tot = 0.0;
  if (e > s) {
    const int64_t m0 = (s - base) / chunk, m1 = (e - 1 - base) / chunk;
    for (int64_t m = m0; m <= m1; ++m)
      tot = __dadd_rn(tot, part[((key - b * K) + b * (K + ns) + m) * d + f]);
  }
  double* o = sums + key * d + f;
  *o = accumulate ? __dadd_rn(*o, tot) : tot;
}

// Spans beyond what the piece slots hold (update_chunk << N / 4096): one warp
// per (key, 32 features) walks the key's whole run, closing a segment at every
// span boundary (same order, no partial storage).
template <int U>
__global__ void __launch_bounds__(256)
    k_segsum_serial(const double* __restrict__ X, const int32_t* __restrict__ order,
                    const int64_t* __restrict__ off, int64_t BK, int64_t K, int d, int fgs,
                    int64_t chunk, double* __restrict__ sums, int accumulate) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= BK * fgs) return;
  const int64_t key = warp / fgs;
  const int f = (int)(warp - key * fgs) * 32 + lane;
  const bool act = f < d;
  const int64_t b = key / K;
  const int64_t s = off[key], e = off[key + 1], base = off[b * K];
  int64_t nb = base + ((s - base) / chunk + 1) * chunk;  // first span start after s
  double tot = 0.0, acc = 0.0;
  for (int64_t p0 = s; p0 < e; p0 += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = p0 + u;
      const int64_t row = p < e ? (int64_t)__ldg(order + p) : 0;
      v[u] = (act && p < e) ? __ldg(X + row * d + f) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = p0 + u;
      if (p < e) {
        if (p == nb) {  // span boundary: merge the finished segment
          tot = __dadd_rn(tot, acc);
          acc = 0.0;
          nb += chunk;
        }
        acc = __dadd_rn(acc, v[u]);
      }
    }
  }
  tot = __dadd_rn(tot, acc);
  if (act) {
    double* o = sums + key * d + f;
    *o = accumulate ? __dadd_rn(*o, tot) : tot;
  }
}


static bool segsum_f64_serial() {
  static int v = -1;  // FK_SEGSUM_F64=parallel: the slice-parallel k_segsum for f64 (A/B)
  if (v < 0) {
    const char* e = getenv("FK_SEGSUM_F64");
    v = (e && e[0] == 'p') ? 0 : 1;
  }
  return v == 1;
}

template <typename T, typename A>
static cudaError_t dispatch_segsum(const void* X, const UpdateWs& w, int64_t BK, int64_t P, int64_t d,
                                   double* sums, int num_sms, cudaStream_t s, const int32_t* ids,
                                   int64_t N, int64_t K, int accumulate, bool clear_table) {
  const int th = 256;
  const int64_t L = segsum_slice(P, BK, num_sms, sizeof(T) == 2 ? DT_BF16 : sizeof(T) == 4 ? DT_F32 : DT_F64);
  const int64_t warps = (P + L - 1) / L;
  const unsigned grid = (unsigned)((warps * 32 + th - 1) / th);
  const int64_t row_bytes = d * (int64_t)sizeof(T);
  const bool vec_ok = (row_bytes % 16) == 0;
  const int64_t nvec = row_bytes / 16;  // 16-byte vectors per row
  const T* x = (const T*)X;
  const SegMerge mg{w.part, w.arrive, L, d, clear_table ? w.table : nullptr, clear_table ? w.zero_n : 0};
  const bool seq_env = !segsum_chained(P, BK);
#define FK_SEG2(LPR, VPL, U, U2)                                                                        \
  do {                                                                                                  \
    if (seq_env)                                                                                        \
      launch_maybe_pdl(k_segsum<T, A, LPR, VPL, U>, grid, th, 0, s, x, w.order, w.off, BK, L, d, sums, ids, N, K, mg); \
    else                                                                                                \
      launch_maybe_pdl(k_segsum2<T, A, LPR, VPL, U2>, grid, th, 0, s, x, w.order, w.off, BK, L, d, sums, ids, N, K,   \
                       mg, accumulate);                                \
  } while (0)
  // k_segsum2 keeps 6 row steps where k_segsum had 8 (64 registers, no spills)
#define FK_SEG(LPR, VPL, U) FK_SEG2(LPR, VPL, U, (U > 6 ? 6 : U))
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
        k_segsum_generic<T><<<grid, th, 0, s>>>(x, w.order, w.off, BK, L, d, sums, mg);
    }
  } else {
    k_segsum_generic<T><<<grid, th, 0, s>>>(x, w.order, w.off, BK, L, d, sums, mg);
  }
#undef FK_SEG
#undef FK_SEG2
  return cudaGetLastError();
}

static bool scatter_is_warp(int64_t K) {
  static int radix_env = -1;  // FK_SCATTER_RADIX=1: the block radix sort for every K (A/B)
  if (radix_env < 0) {
    const char* e = getenv("FK_SCATTER_RADIX");
    radix_env = (e && e[0] == '1') ? 1 : 0;
  }
  return K <= SW_KMAX && !radix_env;
}

// The stable scatter.  The warp-table kernel also does the key scan (off,
// counts, merges); the radix kernel needs k_scan to have run.
static cudaError_t launch_scatter_stable(const int32_t* ids, int64_t B, int64_t N, int64_t K,
                                         int64_t bpb, const UpdateWs& w, int64_t chunk, int accumulate,
                                         int64_t* counts, int64_t* merges, cudaStream_t s,
                                         double* zero_sums = nullptr, int64_t zero_n = 0,
                                         bool zero_arrive = false) {
  int bits = 1;
  while (bits < 31 && ((K - 1) >> bits) != 0) ++bits;
  const int np = (bits + 7) / 8;
  const int last_bits = bits - 8 * (np - 1);
  static int match_env = -1;  // FK_SCATTER_MATCH=1: match.any instead of per-bit ballots (A/B)
  if (match_env < 0) {
    const char* e = getenv("FK_SCATTER_MATCH");
    match_env = (e && e[0] == '1') ? 1 : 0;
  }
  const unsigned blocks = (unsigned)(B * bpb);
  if (scatter_is_warp(K)) {
    // warp-table budget per block: 64 KB, or 96 KB from K = 2048 on (K = 4096:
    // 8 warps per block instead of 4; config 3 459.6 vs 469.9 us, configs 2
    // and 4 are slower with wider tables, profiles/r02_ab_sw_table.txt);
    // FK_SW_TABLE_KB overrides (A/B)
    static int tab_env = -2;
    if (tab_env == -2) {
      const char* e = getenv("FK_SW_TABLE_KB");
      tab_env = e ? atoi(e) * 1024 : -1;
      if (e && tab_env < 4096) tab_env = -1;
    }
    const int tab_bytes = tab_env > 0 ? tab_env : (K >= 2048 ? 96 * 1024 : SW_TABLE_BYTES);
    // FK_SCATTER_RANK=sort: bitonic (id, lane) ranks instead of returning
    // atomics (A/B: config 3 update 521 vs 465 us, profiles/r02_ab_rank.txt)
    static int rank_sort = -1;
    if (rank_sort < 0) {
      const char* e = getenv("FK_SCATTER_RANK");
      rank_sort = (e && e[0] == 's') ? 1 : 0;
    }
    int W = 32;
    while (W > 1 && (int64_t)W * (K + 2) * 2 > tab_bytes) W >>= 1;
    const bool alias = (int64_t)W * (K + 2) * 2 >= K * 4;
    const size_t smem = (size_t)((W * (K + 2) * 2 + 15) & ~15) + (size_t)K * (alias ? 4 : 8);
    const bool cols = bpb <= SW_COLS_BPB;
#define FK_SW2(WV, CV)                                                                             \
  do {                                                                                             \
    static bool attr_set[64] = {};                                                                 \
    int dev = 0;                                                                                   \
    cudaGetDevice(&dev);                                                                           \
    if (!attr_set[dev & 63]) { /* the largest table + bases */                                     \
      cudaFuncSetAttribute(k_scatter_warp<WV, CV>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                           220 * 1024);                                                            \
      attr_set[dev & 63] = true;                                                                   \
    }                                                                                              \
    k_scatter_warp<WV, CV><<<blocks, WV * 32, smem, s>>>(ids, N, K, (int)bpb, w.table, w.hist,     \
                                                         w.inval, B, chunk, accumulate, w.off,     \
                                                         counts, merges, w.order, rank_sort,       \
                                                         zero_sums, zero_n,                        \
                                                         zero_arrive ? w.arrive : nullptr,         \
                                                         zero_arrive ? B * K : 0);                 \
  } while (0)
#define FK_SW(WV)        \
  do {                   \
    if (cols)            \
      FK_SW2(WV, true);  \
    else                 \
      FK_SW2(WV, false); \
  } while (0)
    switch (W) {
      case 32: FK_SW(32); break;
      case 16: FK_SW(16); break;
      case 8: FK_SW(8); break;
      case 4: FK_SW(4); break;
      case 2: FK_SW(2); break;
      default: FK_SW(1);
    }
#undef FK_SW
#undef FK_SW2
    return cudaGetLastError();
  }
  const bool sb = K <= SD_KSMEM;
  const size_t smem = sb ? SD_SMEM_BASES : SD_SMEM;
#define FK_SCAT(NPV, SB, MA)                                                                       \
  do {                                                                                             \
    static bool attr_set[64] = {};                                                                 \
    int dev = 0;                                                                                   \
    cudaGetDevice(&dev);                                                                           \
    if (!attr_set[dev & 63]) { /* one-time per device: keeps graph capture free of it */           \
      cudaFuncSetAttribute(k_scatter_stable<NPV, SB, MA>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)SD_SMEM_BASES);                                                    \
      attr_set[dev & 63] = true;                                                                   \
    }                                                                                              \
    k_scatter_stable<NPV, SB, MA><<<blocks, SD_T, smem, s>>>(ids, N, K, (int)bpb, last_bits,       \
                                                              w.table, w.off, w.order);            \
  } while (0)
#define FK_SCAT_NP(SB, MA)              \
  switch (np) {                         \
    case 1: FK_SCAT(1, SB, MA); break;  \
    case 2: FK_SCAT(2, SB, MA); break;  \
    case 3: FK_SCAT(3, SB, MA); break;  \
    default: FK_SCAT(4, SB, MA);        \
  }
  if (sb) {
    if (match_env) FK_SCAT_NP(true, true) else FK_SCAT_NP(true, false)
  } else {
    if (match_env) FK_SCAT_NP(false, true) else FK_SCAT_NP(false, false)
  }
#undef FK_SCAT_NP
#undef FK_SCAT
  return cudaGetLastError();
}

// After k_hist: the column prefix (k_colscan, unless the warp scatter does it
// itself), the key scan (inside the warp scatter; k_scan for the radix one)
// and the stable scatter.
static cudaError_t launch_sort_passes(const int32_t* ids, int64_t B, int64_t N, int64_t K, int64_t bpb,
                                      const UpdateWs& w, int64_t chunk, int accumulate, int64_t* counts,
                                      int64_t* merges, cudaStream_t s, double* zero_sums = nullptr,
                                      int64_t zero_n = 0, bool zero_arrive = false) {
  const bool warp = scatter_is_warp(K);
  if (!(warp && bpb <= SW_COLS_BPB)) {
    const int64_t ktiles = (K + 31) / 32;
    k_colscan<<<(unsigned)(B * ktiles), dim3(32, 32), 0, s>>>(w.table, K, (int)bpb, ktiles, w.hist);
  }
  if (!warp) k_scan<<<(unsigned)B, 1024, 0, s>>>(w.hist, B, N, K, chunk, accumulate, w.off, counts, merges);
  return launch_scatter_stable(ids, B, N, K, bpb, w, chunk, accumulate, counts, merges, s, zero_sums,
                               zero_n, zero_arrive);
}

// The stable argsort alone (argsort_assignments, sort_inverse.py:67-78):
// order_out (B*N int32 flat point indices, valid ids only) and the key offsets
// off_out (B*K+1 int64); the workspace is fk_update's for d = 1.
cudaError_t launch_argsort(const int32_t* ids, int64_t B, int64_t N, int64_t K, int32_t* order_out,
                           int64_t* off_out, void* ws, int num_sms, cudaStream_t s) {
  const int sms = num_sms < kMaxSms ? num_sms : kMaxSms;
  UpdateWs w;
  update_ws_layout(DT_F32, B, N, K, 1, sms, ws, &w);
  w.order = order_out;
  w.off = off_out;
  const int64_t bpb = update_bpb(B, N, K, sms);
  cudaError_t e;
  const bool smem_keys = K <= HIST_SMEM_KEYS;
  if (!smem_keys && (e = cudaMemsetAsync(w.table, 0, (size_t)B * bpb * K * 4, s)) != cudaSuccess)
    return e;
  k_hist<<<(unsigned)(B * bpb), 1024, smem_keys ? K * 4 : 0, s>>>(ids, N, K, (int)bpb, w.table, nullptr,
                                                                  0, nullptr, 0, w.inval);
  return launch_sort_passes(ids, B, N, K, bpb, w, N, 0, nullptr, nullptr, s);
}

// The block histogram table inside an update workspace, for the assign to
// build (fk_assign_hist): table (B * bpb rows of K int32), inval (B * bpb),
// blocks per batch element and points per block.  False where the fold is not
// offered (the radix scatter, K > SW_KMAX).
bool update_hist_slots(int dt, int64_t B, int64_t N, int64_t K, int64_t d, int num_sms, void* ws,
                       int32_t** table, int32_t** inval, int64_t* bpb_out, int64_t* per_out,
                       int64_t* words) {
  if (!scatter_is_warp(K)) return false;
  const int sms = num_sms < kMaxSms ? num_sms : kMaxSms;
  UpdateWs w;
  update_ws_layout(dt, B, N, K, d, sms, ws, &w);
  const int64_t bpb = update_bpb(B, N, K, sms);
  *table = w.table;
  *inval = w.inval;
  *bpb_out = bpb;
  *per_out = (N + bpb - 1) / bpb;
  *words = w.zero_n;
  return true;
}

cudaError_t launch_update(int dt, const void* X, const int32_t* ids, int64_t B, int64_t N,
                          int64_t K, int64_t d, int64_t chunk, int accumulate, double* sums,
                          int64_t* counts, int64_t* merges, void* ws, int num_sms,
                          cudaStream_t s, int prehist) {
  const int64_t BK = B * K, P = B * N;
  const int sms = num_sms < kMaxSms ? num_sms : kMaxSms;
  UpdateWs w;
  update_ws_layout(dt, B, N, K, d, sms, ws, &w);
  const int64_t bpb = update_bpb(B, N, K, sms);
  const unsigned blocks = (unsigned)(B * bpb);
  cudaError_t e;
  const int64_t ch = chunk < 1 ? 1 : (chunk > N ? N : chunk);
  if (prehist) {
    // the assign built the block table (fk_assign_hist): no k_hist; the
    // scatter clears the sums and arrival counters, k_segsum the table
    if (!scatter_is_warp(K) || dt == DT_F64) return cudaErrorInvalidValue;
    if ((e = launch_sort_passes(ids, B, N, K, bpb, w, ch, accumulate, counts, merges, s,
                                accumulate ? nullptr : sums, BK * d, true)) != cudaSuccess)
      return e;
  } else {
    const bool smem_keys = K <= HIST_SMEM_KEYS;
    if (!smem_keys && (e = cudaMemsetAsync(w.table, 0, (size_t)B * bpb * K * 4, s)) != cudaSuccess)
      return e;
    // sums are cleared inside k_hist unless accumulating; so are the arrival counters
    k_hist<<<blocks, 1024, smem_keys ? K * 4 : 0, s>>>(ids, N, K, (int)bpb, w.table,
                                                       accumulate ? nullptr : sums, BK * d, w.arrive, BK,
                                                       w.inval);
    if ((e = launch_sort_passes(ids, B, N, K, bpb, w, ch, accumulate, counts, merges, s)) != cudaSuccess)
      return e;
  }
  switch (dt) {
    case DT_BF16: return dispatch_segsum<__nv_bfloat16, float>(X, w, BK, P, d, sums, sms, s, ids, N, K, accumulate, prehist != 0);
    case DT_F16: return dispatch_segsum<__half, float>(X, w, BK, P, d, sums, sms, s, ids, N, K, accumulate, prehist != 0);
    case DT_F32: return dispatch_segsum<float, double>(X, w, BK, P, d, sums, sms, s, ids, N, K, accumulate, prehist != 0);
    default:
      if (segsum_f64_serial()) {
        const int fgs = (int)((d + 31) / 32);
        const int64_t ns = (N + ch - 1) / ch;  // spans per batch element
        if (ns <= kF64MaxSpans) {
          // piece warps per key: about the spans an average run touches (a
          // longer run loops), so the grid stays near one warp per piece
          int64_t jwe = (N + K * ch - 1) / (K * ch) + 1;
          if (jwe > ns) jwe = ns;
          const int jw = (int)(jwe < 1 ? 1 : (jwe > 64 ? 64 : jwe));
          const int64_t threads = BK * jw * fgs * 32;
          k_seg_pieces<16><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
              (const double*)X, w.order, w.off, BK, K, (int)d, fgs, ch, ns, jw, w.part);
          k_seg_fold<<<(unsigned)((BK * d + 255) / 256), 256, 0, s>>>(w.off, BK, K, (int)d, ch, ns,
                                                                    w.part, sums, accumulate);
        } else {
          const int64_t threads = BK * fgs * 32;
          k_segsum_serial<16><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
              (const double*)X, w.order, w.off, BK, K, (int)d, fgs, ch, sums, accumulate);
        }
        return cudaGetLastError();
      }
      return dispatch_segsum<double, double>(X, w, BK, P, d, sums, sms, s, ids, N, K, accumulate, prehist != 0);
  }
}

// ----------------------------------------------------------------- normalize
constexpr int NORM_RW = 4;  // centroid rows per warp in k_normalize

FK_DEV float op_to_f32(float v) { return v; }
FK_DEV float op_to_f32(double v) { return (float)v; }
FK_DEV float op_to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
FK_DEV float op_to_f32(__half v) { return __half2float(v); }

// c = fl(s / n) per cluster (empty clusters keep prev bitwise), the rounded MMA
// operand, the empty mask and max ||c_new - c_prev||^2 -- and, for a bf16/fp16
// operand, the tensor-core bias operand of the NEXT assign: the [hi, mid, lo]
// bf16 split of ||c||^2 / 2 of the rounded row, with exactly the arithmetic of
// k_cn_ext (lane-strided fmaf over the columns in increasing order, then an
// xor-shuffle tree), so precomputing it here leaves the assignment bitwise
// unchanged and saves the assign its own pass over C.
// The end of a single-device iteration in the same launch (TAIL): the blocks
// also compute the objective partials (k_obj_partial's blocks and tree, so the
// same doubles) and the last block to finish runs k_loop_tail's work
// (objective, history row, flags, cleared accumulators).
struct TailArgs {
  const void* mind;
  int mind_f64;
  int64_t B, N, nblk;
  double* part;
  double* obj;
  double* hist;
  int64_t* hist_it;
  int32_t* changed;
  int64_t* merges;
  double* flags;
  unsigned int* counter;
  int obj_ready;  // obj[] already holds the objective (f64 min_dists: numpy's pairwise tree)
  int64_t norm_blocks;  // blocks that normalize; the rest sum objective partials
};

// Objective partials: numpy's order for np.sum(m, dtype=float64) of an f32
// row (np_pairwise_block, fk_common.cuh): one partial per 8192-element buffer,
// folded in buffer order from 0.0 (obj_fold).  f64 rows: launch_pairwise_total.
constexpr int OBJ_BLOCK_N = kNpBuf;
constexpr int TAIL_STAGE = 4096;  // objective partials the last block stages in shared memory

// obj = ((0 + part[0]) + part[1]) + ... (numpy's running sum over its buffers)
FK_DEV double obj_fold(const double* part, int64_t n) {
  double acc = 0.0;
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {  // loads ahead of the serial adds
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = part[i + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
  }
  for (; i < n; ++i) acc = __dadd_rn(acc, part[i]);
  return acc;
}

template <typename TM, typename TO, bool TAIL = false>
__global__ void __launch_bounds__(256)
    k_normalize(const double* __restrict__ sums, const int64_t* __restrict__ counts,
                const TM* __restrict__ prev, TM* __restrict__ out, TO* __restrict__ operand,
                uint8_t* __restrict__ empty, double* max_shift2, int64_t BK, int64_t d,
                __nv_bfloat16* __restrict__ bias, int64_t K, int64_t kpad, TailArgs ta = TailArgs{}) {
  // TAIL: blocks [0, norm_blocks) normalize, the others sum objective
  // partials, concurrently (one block doing both would serialize them)
  pdl_wait();
  if (!TAIL || blockIdx.x < ta.norm_blocks) {
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
    float nrm[RW];
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      cnt[q] = row0 + q < BK ? counts[row0 + q] : 0;
      sh[q] = 0.0;
      nrm[q] = 0.f;
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
            if (operand) {
              const TO ov = (TO)(float)nv;
              operand[o] = ov;
              const float f = op_to_f32(ov);
              nrm[q] = fmaf(f, f, nrm[q]);
            }
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
    if (bias) {
#pragma unroll
      for (int q = 0; q < RW; ++q) {
        float acc = nrm[q];
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (row0 + q < BK && lane < 16) {
          const int64_t b = (row0 + q) / K, k = row0 + q - b * K;
          const float v = 0.5f * acc;
          const __nv_bfloat16 hi = __float2bfloat16_rn(v);
          const float r1 = v - __bfloat162float(hi);
          const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
          const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
          bias[(b * kpad + k) * 16 + lane] =
              lane == 0 ? hi : lane == 1 ? mid : lane == 2 ? lo : __float2bfloat16(0.f);
        }
      }
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
  if constexpr (TAIL) {
    __shared__ NpScratch nps;
    const int t = threadIdx.x;
    const int64_t nob_blocks = (int64_t)gridDim.x - ta.norm_blocks;
    for (int64_t ob = (int64_t)blockIdx.x - ta.norm_blocks; !ta.obj_ready && ob >= 0 && ob < ta.B * ta.nblk;
         ob += nob_blocks) {  // k_obj_partial
      const int64_t b = ob / ta.nblk, blk = ob - b * ta.nblk;
      const int64_t lo = blk * OBJ_BLOCK_N;
      const int64_t hi = (lo + OBJ_BLOCK_N < ta.N) ? lo + OBJ_BLOCK_N : ta.N;
      const double v =
          ta.mind_f64 ? np_pairwise_block(reinterpret_cast<const double*>(ta.mind) + b * ta.N + lo,
                                          (int)(hi - lo), nps)
                      : np_pairwise_block(reinterpret_cast<const float*>(ta.mind) + b * ta.N + lo,
                                          (int)(hi - lo), nps);
      if (t == 0) ta.part[ob] = v;
    }
    // the last block to arrive finishes the iteration
    __shared__ int s_last;
    __shared__ double tstage[TAIL_STAGE];
    // what the last block reads from this one (the partials, by thread 0;
    // the shift by atomics) is published by thread 0's fence alone: a fence in
    // every thread would wait for all of the block's normalize stores
    __syncthreads();
    if (t == 0) {
      __threadfence();
      s_last = atomicAdd(ta.counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      const int64_t row = ta.hist ? __ldcg(ta.hist_it) : 0;
      // every partial fetched in one round into shared memory when they fit
      // (B * nblk <= TAIL_STAGE: 64 batch elements of 128K points), instead of
      // one dependent L2 round trip per batch element a warp walks
      const int64_t np = ta.obj_ready ? 0 : ta.B * ta.nblk;
      const bool staged = np <= TAIL_STAGE;
      if (staged) {
        for (int64_t i = t; i < np; i += 256) tstage[i] = __ldcg(ta.part + i);
        __syncthreads();
      }
      for (int64_t b = t; b < ta.B; b += 256) {  // one thread per batch element
        double x;
        if (ta.obj_ready) {
          x = __ldcg(ta.obj + b);
        } else {
          x = staged ? obj_fold(tstage + b * ta.nblk, ta.nblk) : 0.0;
          if (!staged)
            for (int64_t i = 0; i < ta.nblk; ++i) x = __dadd_rn(x, __ldcg(ta.part + b * ta.nblk + i));
          ta.obj[b] = x;
        }
        if (ta.hist) ta.hist[row * ta.B + b] = x;
      }
      __syncthreads();
      if (t == 0) {
        if (ta.hist) *ta.hist_it = row + 1;
        ta.flags[0] = (double)__ldcg(ta.changed);
        ta.flags[1] = __ldcg(max_shift2);
        ta.flags[2] = (double)__ldcg(ta.merges);
        *ta.changed = 0;
        *max_shift2 = 0.0;
        *ta.merges = 0;
        *ta.counter = 0u;
      }
    }
  }
}

template <typename TM>
static cudaError_t norm_dispatch(int operand_dt, const double* sums, const int64_t* counts,
                                 const void* prev, void* out, void* operand_out, uint8_t* empty,
                                 double* ms2, int64_t BK, int64_t d, void* bias, int64_t K,
                                 int64_t kpad, cudaStream_t s) {
  const int th = 256;
  const int64_t rows_per_block = (th / 32) * NORM_RW;
  const unsigned grid = (unsigned)((BK + rows_per_block - 1) / rows_per_block);
  const TM* pv = (const TM*)prev;
  TM* ov = (TM*)out;
  __nv_bfloat16* bz = (__nv_bfloat16*)bias;
  if (!operand_out)
    k_normalize<TM, float><<<grid, th, 0, s>>>(sums, counts, pv, ov, nullptr, empty, ms2, BK, d,
                                               nullptr, K, kpad);
  else if (operand_dt == DT_BF16)
    k_normalize<TM, __nv_bfloat16><<<grid, th, 0, s>>>(sums, counts, pv, ov, (__nv_bfloat16*)operand_out,
                                                       empty, ms2, BK, d, bz, K, kpad);
  else if (operand_dt == DT_F16)
    k_normalize<TM, __half><<<grid, th, 0, s>>>(sums, counts, pv, ov, (__half*)operand_out, empty,
                                               ms2, BK, d, bz, K, kpad);
  else if (operand_dt == DT_F32)
    k_normalize<TM, float><<<grid, th, 0, s>>>(sums, counts, pv, ov, (float*)operand_out, empty,
                                              ms2, BK, d, nullptr, K, kpad);
  else
    k_normalize<TM, double><<<grid, th, 0, s>>>(sums, counts, pv, ov, (double*)operand_out, empty,
                                               ms2, BK, d, nullptr, K, kpad);
  return cudaGetLastError();
}

template <typename TM>
static cudaError_t norm_tail_dispatch(int operand_dt, const double* sums, const int64_t* counts,
                                      const void* prev, void* out, void* operand_out, uint8_t* empty,
                                      double* ms2, int64_t BK, int64_t d, void* bias, int64_t K,
                                      int64_t kpad, const TailArgs& ta_in, cudaStream_t s) {
  const int th = 256;
  const int64_t rows_per_block = (th / 32) * NORM_RW;
  TailArgs ta = ta_in;
  ta.norm_blocks = (BK + rows_per_block - 1) / rows_per_block;
  // + one block per objective partial (up to 1024; they loop beyond)
  const int64_t nob = ta.obj_ready ? 0 : (ta.B * ta.nblk < 1024 ? ta.B * ta.nblk : 1024);
  const unsigned grid = (unsigned)(ta.norm_blocks + nob);
  const TM* pv = (const TM*)prev;
  TM* ov = (TM*)out;
  __nv_bfloat16* bz = (__nv_bfloat16*)bias;
  if (!operand_out)
    launch_maybe_pdl(k_normalize<TM, float, true>, grid, th, 0, s, sums, counts, pv, ov, (float*)nullptr,
                     empty, ms2, BK, d, (__nv_bfloat16*)nullptr, K, kpad, ta);
  else if (operand_dt == DT_BF16)
    launch_maybe_pdl(k_normalize<TM, __nv_bfloat16, true>, grid, th, 0, s, sums, counts, pv, ov,
                     (__nv_bfloat16*)operand_out, empty, ms2, BK, d, bz, K, kpad, ta);
  else if (operand_dt == DT_F16)
    launch_maybe_pdl(k_normalize<TM, __half, true>, grid, th, 0, s, sums, counts, pv, ov,
                     (__half*)operand_out, empty, ms2, BK, d, bz, K, kpad, ta);
  else if (operand_dt == DT_F32)
    launch_maybe_pdl(k_normalize<TM, float, true>, grid, th, 0, s, sums, counts, pv, ov,
                     (float*)operand_out, empty, ms2, BK, d, (__nv_bfloat16*)nullptr, K, kpad, ta);
  else
    launch_maybe_pdl(k_normalize<TM, double, true>, grid, th, 0, s, sums, counts, pv, ov,
                     (double*)operand_out, empty, ms2, BK, d, (__nv_bfloat16*)nullptr, K, kpad, ta);
  return cudaGetLastError();
}

cudaError_t launch_normalize_tail(int master_dt, const double* sums, const int64_t* counts,
                                  const void* prev, void* out, int operand_dt, void* operand_out,
                                  uint8_t* empty_mask, double* max_shift2, int64_t B, int64_t K,
                                  int64_t d, void* bias_out, int64_t bias_kpad, int mind_f64,
                                  const void* mind, int64_t N, double* part, double* obj,
                                  double* hist, int64_t* hist_it, int32_t* changed,
                                  int64_t* merges, double* flags, unsigned int* counter,
                                  int num_sms, cudaStream_t s) {
  // More objective blocks (8192-point buffers) than one wave of the
  // normalize kernel's register slots (2 per SM): the objective blocks would
  // queue behind each other inside the one launch -- three launches instead
  // (normalize, partials, loop tail; graph-replayed, profiles/r02_ab_tail.txt:
  // config 3 (1024 buffers) 20.3 vs 22.0 us, B=8 x 1M points 15.2 vs 15.9 us;
  // the one launch wins at config 2 (128 buffers) 9.5 vs 11.7 us and ties at
  // config 4, 14.0 vs 13.9-14.6 us).  FK_TAIL=fused|split overrides (A/B).
  static int tail_env = -2;
  if (tail_env == -2) {
    const char* e = getenv("FK_TAIL");
    tail_env = !e ? -1 : (e[0] == 'f' ? 1 : e[0] == 's' ? 0 : -1);
  }
  if (!mind_f64) {
    const int64_t nblk = (N + OBJ_BLOCK_N - 1) / OBJ_BLOCK_N;
    const bool split = tail_env >= 0 ? tail_env == 0 : B * nblk > 2 * (int64_t)num_sms;
    if (split) {
      cudaError_t e = launch_normalize(master_dt, sums, counts, prev, out, operand_dt, operand_out, empty_mask,
                                       max_shift2, B, K, d, bias_out, bias_kpad, s);
      if (e == cudaSuccess) e = launch_objective_partials(0, mind, B, N, part, s);
      if (e == cudaSuccess)
        e = launch_loop_tail(part, B, N, obj, hist, hist_it, changed, max_shift2, merges, flags, s);
      return e;
    }
  }
  TailArgs ta;
  ta.mind = mind;
  ta.mind_f64 = mind_f64;
  ta.B = B;
  ta.N = N;
  ta.nblk = (N + OBJ_BLOCK_N - 1) / OBJ_BLOCK_N;
  ta.part = part;
  ta.obj = obj;
  ta.hist = hist;
  ta.hist_it = hist_it;
  ta.changed = changed;
  ta.merges = merges;
  ta.flags = flags;
  ta.counter = counter;
  ta.obj_ready = 0;
  if (mind_f64 && launch_pairwise_total((const double*)mind, B, N, obj, part, s) == cudaSuccess)
    ta.obj_ready = 1;  // part is the objective workspace (objective_workspace_bytes)
  (void)cudaGetLastError();
  if (master_dt == DT_F64)
    return norm_tail_dispatch<double>(operand_dt, sums, counts, prev, out, operand_out, empty_mask,
                                      max_shift2, B * K, d, bias_out, K, bias_kpad, ta, s);
  return norm_tail_dispatch<float>(operand_dt, sums, counts, prev, out, operand_out, empty_mask,
                                   max_shift2, B * K, d, bias_out, K, bias_kpad, ta, s);
}

cudaError_t launch_normalize(int master_dt, const double* sums, const int64_t* counts,
                             const void* prev, void* out, int operand_dt, void* operand_out,
                             uint8_t* empty_mask, double* max_shift2, int64_t B, int64_t K,
                             int64_t d, void* bias_out, int64_t bias_kpad, cudaStream_t s) {
  if (master_dt == DT_F64)
    return norm_dispatch<double>(operand_dt, sums, counts, prev, out, operand_out, empty_mask,
                                 max_shift2, B * K, d, bias_out, K, bias_kpad, s);
  return norm_dispatch<float>(operand_dt, sums, counts, prev, out, operand_out, empty_mask,
                              max_shift2, B * K, d, bias_out, K, bias_kpad, s);
}

// ----------------------------------------------------------------- objective
// Deterministic two-level reduction (fixed 8192-element blocks, fixed trees).
// For float32 min_dists every float64 partial sum is exact in practice, so
// the result equals numpy's np.sum(m, dtype=float64) bit for bit; for
// float64 data the summation order differs from numpy's pairwise tree.
constexpr int OBJ_BLOCK = OBJ_BLOCK_N;

template <typename T>
__global__ void __launch_bounds__(256) k_obj_partial(const T* __restrict__ m, int64_t B, int64_t N,
                                                     int64_t nblk, double* part) {
  __shared__ NpScratch nps;
  const int64_t b = blockIdx.y, blk = blockIdx.x;
  const int64_t lo = blk * OBJ_BLOCK;
  const int64_t hi = (lo + OBJ_BLOCK < N) ? lo + OBJ_BLOCK : N;
  const double v = np_pairwise_block(m + b * N + lo, (int)(hi - lo), nps);
  if (threadIdx.x == 0) part[b * nblk + blk] = v;
}

// The buffer partials of every batch element folded in order (one thread per
// batch element, the partials staged in shared memory when they fit).
FK_DEV double obj_fold_staged(const double* __restrict__ part, int64_t b, int64_t nblk, double* stage,
                              bool staged) {
  return staged ? obj_fold(stage + b * nblk, nblk) : obj_fold(part + b * nblk, nblk);
}

__global__ void __launch_bounds__(256) k_obj_final(const double* part, int64_t B, int64_t nblk,
                                                   double* out) {
  __shared__ double stage[TAIL_STAGE];
  const bool staged = B * nblk <= TAIL_STAGE;
  if (staged)
    for (int64_t i = threadIdx.x; i < B * nblk; i += blockDim.x) stage[i] = part[i];
  __syncthreads();
  for (int64_t b = threadIdx.x; b < B; b += blockDim.x) out[b] = obj_fold_staged(part, b, nblk, stage, staged);
}

// End of one device-resident Lloyd iteration, one launch (LloydEngine): the
// objective partials folded in numpy's order into obj[b] and the history row
// hist[(*it) * B + b] (*it advanced: the row index lives on the device, so a
// replayed CUDA graph writes successive rows); flags = [changed, max shift^2,
// merges] for the one host read; the three accumulators cleared for the next
// iteration.
__global__ void __launch_bounds__(256)
    k_loop_tail(const double* __restrict__ part, int64_t B, int64_t nblk, double* __restrict__ obj,
                double* __restrict__ hist, int64_t* __restrict__ hist_it, int32_t* changed,
                double* shift2, int64_t* merges, double* __restrict__ flags) {
  __shared__ double stage[TAIL_STAGE];
  const bool staged = B * nblk <= TAIL_STAGE;
  if (staged)
    for (int64_t i = threadIdx.x; i < B * nblk; i += blockDim.x) stage[i] = part[i];
  __syncthreads();
  const int64_t row = hist ? *hist_it : 0;
  for (int64_t b = threadIdx.x; b < B; b += blockDim.x) {
    const double x = obj_fold_staged(part, b, nblk, stage, staged);
    obj[b] = x;
    if (hist) hist[row * B + b] = x;
  }
  __syncthreads();  // every thread read *hist_it before it moves
  if (threadIdx.x == 0) {
    if (hist) *hist_it = row + 1;
    flags[0] = (double)*changed;
    flags[1] = *shift2;
    flags[2] = (double)*merges;
    *changed = 0;
    *shift2 = 0.0;
    *merges = 0;
  }
}

cudaError_t launch_objective_partials(int mind_is_f64, const void* mind, int64_t B, int64_t N,
                                      double* part, cudaStream_t s) {
  const int64_t nblk = (N + OBJ_BLOCK - 1) / OBJ_BLOCK;
  dim3 grid((unsigned)nblk, (unsigned)B);
  if (mind_is_f64)
    k_obj_partial<double><<<grid, 256, 0, s>>>((const double*)mind, B, N, nblk, part);
  else
    k_obj_partial<float><<<grid, 256, 0, s>>>((const float*)mind, B, N, nblk, part);
  return cudaGetLastError();
}

cudaError_t launch_loop_tail(const double* part, int64_t B, int64_t N, double* obj, double* hist,
                             int64_t* hist_it, int32_t* changed, double* shift2, int64_t* merges,
                             double* flags, cudaStream_t s) {
  const int64_t nblk = (N + OBJ_BLOCK - 1) / OBJ_BLOCK;
  k_loop_tail<<<1, 256, 0, s>>>(part, B, nblk, obj, hist, hist_it, changed, shift2, merges, flags);
  return cudaGetLastError();
}

size_t objective_workspace_bytes(int64_t B, int64_t N) {
  const size_t tree = (size_t)(B * ((N + OBJ_BLOCK - 1) / OBJ_BLOCK)) * 8 + 256;
  const size_t pw = pairwise_total_workspace(B, N);  // f64 min_dists: numpy's pairwise order
  return tree > pw ? tree : pw;
}

cudaError_t launch_objective(int mind_is_f64, const void* mind, int64_t B, int64_t N, double* out,
                             void* ws, cudaStream_t s) {
  // f64 min_dists (f64 data): np.sum's pairwise tree exactly (bitwise); f32
  // min_dists: the fixed two-level tree (every f64 partial of f32 values is
  // exact in practice, so any order gives numpy's double)
  if (mind_is_f64 && launch_pairwise_total((const double*)mind, B, N, out, ws, s) == cudaSuccess)
    return cudaSuccess;
  (void)cudaGetLastError();
  const int64_t nblk = (N + OBJ_BLOCK - 1) / OBJ_BLOCK;
  double* part = (double*)ws;
  dim3 grid((unsigned)nblk, (unsigned)B);
  if (mind_is_f64)
    k_obj_partial<double><<<grid, 256, 0, s>>>((const double*)mind, B, N, nblk, part);
  else
    k_obj_partial<float><<<grid, 256, 0, s>>>((const float*)mind, B, N, nblk, part);
  k_obj_final<<<1, 256, 0, s>>>(part, B, nblk, out);
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

FK_MODULE_ANCHOR(update)

}  // namespace fk
