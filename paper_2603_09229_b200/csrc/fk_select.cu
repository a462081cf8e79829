// fk_select.cu -- device top-E for the reseed_farthest policy.
//
// Replaces the reference's _farthest_order / _FarthestTracker (pipeline.py:76-89,
// 283-309): the E points farthest from their assigned centroid, ordered by
// distance descending and, on equal distances, by point index ascending
// (np.lexsort((arange, -mind))).
//
// Every point gets a unique 96-bit key  (f64 bits of its distance) << 32 |
// (2^32 - 1 - index):  a larger key is an earlier point of the reference's
// order.  A most-significant-digit radix select over the 12 key bytes
// (k_sel_hist: one shared-memory histogram of the next byte among the points
// that match the prefix found so far; k_sel_pick: one block picks the byte
// that holds the E-th largest key) finds T, the E-th largest key; exactly E
// points have key >= T.  k_sel_collect gathers them and k_sel_sort orders them
// with a bitonic sort in shared memory.  No host round trip, no sort of all N.
#include "fk_common.cuh"
#include "fk_kernels.h"

namespace fk {

constexpr int SEL_T = 256;
constexpr int SEL_EMAX = 8192;  // E handled by the in-shared-memory final sort

struct SelState {
  unsigned long long pre_hi;   // key bits 95..32 found so far
  unsigned long long mask_hi;
  uint32_t pre_lo, mask_lo;    // key bits 31..0
  long long remaining;         // how many of the E are still to be placed at/below the prefix
  int count;                   // collected points
  int pad;
};

FK_DEV unsigned long long dist_key(float v) { return (unsigned long long)__double_as_longlong((double)v); }
FK_DEV unsigned long long dist_key(double v) { return (unsigned long long)__double_as_longlong(v); }

// byte `pos` (0 = most significant) of the 96-bit key (hi: 64 bits, lo: 32 bits)
FK_DEV uint32_t key_byte(unsigned long long hi, uint32_t lo, int pos) {
  return pos < 8 ? (uint32_t)(hi >> (56 - 8 * pos)) & 0xffu : (lo >> (24 - 8 * (pos - 8))) & 0xffu;
}

template <typename T>
__global__ void __launch_bounds__(SEL_T)
    k_sel_hist(const T* __restrict__ m, int64_t N, int pos, const SelState* __restrict__ st,
               uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  const int64_t b = blockIdx.y;
  h[threadIdx.x] = 0;
  __syncthreads();
  const SelState s = st[b];
  for (int64_t i = blockIdx.x * (int64_t)SEL_T + threadIdx.x; i < N; i += (int64_t)gridDim.x * SEL_T) {
    const unsigned long long hi = dist_key(m[b * N + i]);
    const uint32_t lo = 0xffffffffu - (uint32_t)i;
    if ((hi & s.mask_hi) == s.pre_hi && (lo & s.mask_lo) == s.pre_lo)
      atomicAdd(&h[key_byte(hi, lo, pos)], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&hist[b * 256 + threadIdx.x], h[threadIdx.x]);
}

// one block per batch element: the byte value that holds the remaining-th
// largest key among the prefix matches; clears the histogram for the next pass
__global__ void __launch_bounds__(256) k_sel_pick(int pos, SelState* st, uint32_t* hist) {
  __shared__ uint32_t c[256];
  __shared__ int s_digit;
  __shared__ long long s_above;
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x;
  c[t] = hist[b * 256 + t];
  hist[b * 256 + t] = 0;
  __syncthreads();
  if (t == 0) {
    const long long want = st[b].remaining;
    long long above = 0;
    int dsel = 0;
    for (int dd = 255; dd >= 0; --dd) {  // 256 steps, once per pass
      if (above + (long long)c[dd] >= want) {
        dsel = dd;
        break;
      }
      above += c[dd];
    }
    s_digit = dsel;
    s_above = above;
  }
  __syncthreads();
  if (t == 0) {
    SelState s = st[b];
    s.remaining -= s_above;
    if (pos < 8) {
      s.pre_hi |= (unsigned long long)s_digit << (56 - 8 * pos);
      s.mask_hi |= 0xffull << (56 - 8 * pos);
    } else {
      s.pre_lo |= (uint32_t)s_digit << (24 - 8 * (pos - 8));
      s.mask_lo |= 0xffu << (24 - 8 * (pos - 8));
    }
    st[b] = s;
  }
}

// every point with key >= T (exactly E of them), in any order
template <typename T>
__global__ void __launch_bounds__(SEL_T)
    k_sel_collect(const T* __restrict__ m, int64_t N, SelState* st, int64_t E,
                  unsigned long long* __restrict__ ck_hi, uint32_t* __restrict__ ck_lo) {
  const int64_t b = blockIdx.y;
  const unsigned long long th = st[b].pre_hi;
  const uint32_t tl = st[b].pre_lo;
  for (int64_t i = blockIdx.x * (int64_t)SEL_T + threadIdx.x; i < N; i += (int64_t)gridDim.x * SEL_T) {
    const unsigned long long hi = dist_key(m[b * N + i]);
    const uint32_t lo = 0xffffffffu - (uint32_t)i;
    if (hi > th || (hi == th && lo >= tl)) {
      const int slot = atomicAdd(&st[b].count, 1);
      if (slot < E) {
        ck_hi[b * E + slot] = hi;
        ck_lo[b * E + slot] = lo;
      }
    }
  }
}

// bitonic sort (descending) of the E collected keys in shared memory; the
// point indices come out in the reference's order
__global__ void __launch_bounds__(1024)
    k_sel_sort(int64_t E, const unsigned long long* __restrict__ ck_hi, const uint32_t* __restrict__ ck_lo,
               int64_t* __restrict__ idx_out) {
  extern __shared__ __align__(16) uint8_t sel_sm[];
  int P = 1;
  while (P < E) P <<= 1;
  unsigned long long* kh = reinterpret_cast<unsigned long long*>(sel_sm);
  uint32_t* kl = reinterpret_cast<uint32_t*>(kh + P);
  const int64_t b = blockIdx.x;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    kh[i] = i < E ? ck_hi[b * E + i] : 0ull;
    kl[i] = i < E ? ck_lo[b * E + i] : 0u;  // padding sorts last (key 0)
  }
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool desc = (i & k) == 0;
          const bool gt = kh[l] > kh[i] || (kh[l] == kh[i] && kl[l] > kl[i]);  // key[l] > key[i]
          if (gt == desc) {
            const unsigned long long th = kh[i];
            kh[i] = kh[l];
            kh[l] = th;
            const uint32_t tl = kl[i];
            kl[i] = kl[l];
            kl[l] = tl;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < E; i += blockDim.x) idx_out[b * E + i] = (int64_t)(0xffffffffu - kl[i]);
}

__global__ void k_sel_init(SelState* st, int64_t B, int64_t E) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b < B) st[b].remaining = E;  // the rest was zeroed
}

size_t farthest_workspace_bytes(int64_t B, int64_t E) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  return al((size_t)B * sizeof(SelState)) + al((size_t)B * 256 * 4) + al((size_t)B * E * 8) +
         al((size_t)B * E * 4);
}

cudaError_t launch_farthest(int mind_is_f64, const void* mind, int64_t B, int64_t N, int64_t E,
                            int64_t* idx_out, void* ws, int num_sms, cudaStream_t s) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  uint8_t* w = static_cast<uint8_t*>(ws);
  SelState* st = reinterpret_cast<SelState*>(w);
  w += al((size_t)B * sizeof(SelState));
  uint32_t* hist = reinterpret_cast<uint32_t*>(w);
  w += al((size_t)B * 256 * 4);
  unsigned long long* ck_hi = reinterpret_cast<unsigned long long*>(w);
  w += al((size_t)B * E * 8);
  uint32_t* ck_lo = reinterpret_cast<uint32_t*>(w);
  cudaError_t e;
  if ((e = cudaMemsetAsync(st, 0, (size_t)B * sizeof(SelState), s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(hist, 0, (size_t)B * 256 * 4, s)) != cudaSuccess) return e;
  const int64_t per_sm = 2;
  int64_t nblk = (N + SEL_T * 16 - 1) / (SEL_T * 16);
  if (nblk > (int64_t)num_sms * per_sm) nblk = (int64_t)num_sms * per_sm;
  if (nblk < 1) nblk = 1;
  const dim3 grid((unsigned)nblk, (unsigned)B);
  k_sel_init<<<(unsigned)((B + 255) / 256), 256, 0, s>>>(st, B, E);
  for (int pos = 0; pos < 12; ++pos) {
    if (mind_is_f64)
      k_sel_hist<double><<<grid, SEL_T, 0, s>>>((const double*)mind, N, pos, st, hist);
    else
      k_sel_hist<float><<<grid, SEL_T, 0, s>>>((const float*)mind, N, pos, st, hist);
    k_sel_pick<<<(unsigned)B, 256, 0, s>>>(pos, st, hist);
  }
  if (mind_is_f64)
    k_sel_collect<double><<<grid, SEL_T, 0, s>>>((const double*)mind, N, st, E, ck_hi, ck_lo);
  else
    k_sel_collect<float><<<grid, SEL_T, 0, s>>>((const float*)mind, N, st, E, ck_hi, ck_lo);
  int P = 1;
  while (P < E) P <<= 1;
  const size_t smem = (size_t)P * 12;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaFuncSetAttribute(k_sel_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, SEL_EMAX * 12);
    attr_set[dev & 63] = true;
  }
  k_sel_sort<<<(unsigned)B, 1024, smem, s>>>(E, ck_hi, ck_lo, idx_out);
  return cudaGetLastError();
}

FK_MODULE_ANCHOR(select)

}  // namespace fk
