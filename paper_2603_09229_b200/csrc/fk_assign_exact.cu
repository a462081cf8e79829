// fk_assign_exact.cu -- CUDA-core assignment kernels.
//
// 1. The exact mirror (FK_F32 / FK_F64): reproduces the reference's
//    dot_mode="exact" arithmetic bit for bit (reference
//    _kernels.py:21-45 and :64-82):
//        acc  = sum_{j asc} fl64(fl_T(x_j * c_j))
//        D    = fl_T(max(0, fl64(fl_T(xn + cn)) - 2*acc))
//        a    = lowest k with D == min D   (strict <, ascending k)
//    Every product / add is an explicit round-to-nearest intrinsic, so no FMA
//    contraction can change a bit.
// 2. A CUDA-core fallback for bf16/fp16 data whose row width is outside the
//    tcgen05 buckets (d > 128 or d % 8 != 0): fp32 accumulation, same
//    tie rule.
// 3. Helpers: exact row norms (core.row_norms, core.py:307-318) and the
//    padded fp32 ||c||^2 vector used as the tcgen05 epilogue bias.
#include "fk_common.cuh"
#include "fk_kernels.h"

namespace fk {

template <typename T>
FK_DEV float to_f32(T v);
template <>
FK_DEV float to_f32<float>(float v) { return v; }
template <>
FK_DEV float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
FK_DEV float to_f32<__half>(__half v) { return __half2float(v); }

// ---------------------------------------------------------------- norms
template <typename T>
__global__ void k_row_norms_exact(const T* __restrict__ M, int64_t rows, int64_t d, T* out) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const T* p = M + r * d;
  double acc = 0.0;
  for (int64_t j = 0; j < d; ++j) {
    if constexpr (sizeof(T) == 4) {
      acc = __dadd_rn(acc, (double)__fmul_rn(p[j], p[j]));
    } else {
      acc = __dadd_rn(acc, __dmul_rn(p[j], p[j]));
    }
  }
  out[r] = (T)acc;
}

// Same sums, rows staged through shared memory 128 at a time (coalesced row
// reads; one thread per row keeps the serial ascending-j chain).
template <typename T>
__global__ void __launch_bounds__(128) k_row_norms_staged(const T* __restrict__ M, int64_t rows,
                                                          int64_t d, T* out) {
  constexpr int DC = sizeof(T) == 4 ? 32 : 16;
  __shared__ T ms[DC][129];
  const int tid = threadIdx.x;
  const int64_t row0 = blockIdx.x * (int64_t)128;
  double acc = 0.0;
  for (int64_t j0 = 0; j0 < d; j0 += DC) {
    __syncthreads();
#pragma unroll 8
    for (int e = tid; e < 128 * DC; e += 128) {
      const int r = e / DC, jj = e - r * DC;
      const int64_t gr = row0 + r, j = j0 + jj;
      ms[jj][r] = (gr < rows && j < d) ? M[gr * d + j] : (T)0;
    }
    __syncthreads();
    const int jn = (int)(d - j0 < DC ? d - j0 : DC);
    for (int jj = 0; jj < jn; ++jj) {
      const T v = ms[jj][tid];
      if constexpr (sizeof(T) == 4) {
        acc = __dadd_rn(acc, (double)__fmul_rn(v, v));
      } else {
        acc = __dadd_rn(acc, __dmul_rn(v, v));
      }
    }
  }
  if (row0 + tid < rows) out[row0 + tid] = (T)acc;
}

// ||c||^2 in fp32 for the low-precision paths, padded to kpad with +inf so
// columns beyond K never win the argmin.
template <typename T>
__global__ void k_cn_pad(const T* __restrict__ C, int64_t B, int64_t K, int64_t d, int kpad,
                         float* out, float scale) {
  // one warp per (padded) centroid row; lanes stride over the features
  const int64_t gi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gi >= B * kpad) return;
  const int64_t b = gi / kpad, k = gi - b * kpad;
  if (k >= K) {
    if (lane == 0) out[gi] = __int_as_float(0x7f800000);
    return;
  }
  const T* p = C + (b * K + k) * d;
  float acc = 0.f;
  for (int64_t j = lane; j < d; j += 32) {
    float v = to_f32(p[j]);
    acc = fmaf(v, v, acc);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[gi] = acc * scale;  // scale 0.5 (exact): the TMEM-seed bias ||c||^2/2
}

// Bias operand for the bias-in-GEMM FlashAssign: ||c||^2 / 2 split into three
// bf16 terms (24 significant bits) so that one extra K=16 MMA step against a
// constant ones operand adds it to the accumulator exactly enough.
template <typename T>
__global__ void k_cn_ext_bf16(const T* __restrict__ C, int64_t B, int64_t K, int64_t d,
                              int kpad, __nv_bfloat16* out) {
  const int64_t gi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gi >= B * kpad) return;
  const int64_t b = gi / kpad, k = gi - b * kpad;
  __nv_bfloat16* o = out + gi * 16;
  if (k >= K) {
    if (lane < 16) o[lane] = lane == 0 ? __float2bfloat16(__int_as_float(0x7f800000)) : __float2bfloat16(0.f);
    return;
  }
  const T* p = C + (b * K + k) * d;
  float acc = 0.f;
  for (int64_t j = lane; j < d; j += 32) {
    const float v = to_f32(p[j]);
    acc = fmaf(v, v, acc);
  }
  for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  const float v = 0.5f * acc;
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(hi);
  const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
  const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
  if (lane < 16) o[lane] = lane == 0 ? hi : lane == 1 ? mid : lane == 2 ? lo : __float2bfloat16(0.f);
}

cudaError_t launch_cn_ext(int dt, const void* C, int64_t B, int64_t K, int64_t d, int kpad,
                          void* out, cudaStream_t stream) {
  const int64_t n = B * kpad * 32;
  const int th = 256;
  if (dt == DT_BF16)
    k_cn_ext_bf16<__nv_bfloat16><<<(unsigned)((n + th - 1) / th), th, 0, stream>>>(
        (const __nv_bfloat16*)C, B, K, d, kpad, (__nv_bfloat16*)out);
  else if (dt == DT_F16)
    k_cn_ext_bf16<__half><<<(unsigned)((n + th - 1) / th), th, 0, stream>>>(
        (const __half*)C, B, K, d, kpad, (__nv_bfloat16*)out);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- assign
constexpr int EX_ROWS = 128;  // points per block (one per thread)
constexpr int EX_KT = 16;     // centroids per register tile
constexpr int EX_DC = 32;     // feature chunk staged in smem

// LIST: the block's rows are entries [128 x, 128 x + 128) of the per-batch
// row list (list + b*N, list_cnt[b] entries) -- the rows the certified
// tensor-core path could not decide (fk_assign_split.cu).
template <typename T, bool EXACT, bool LIST = false>
__global__ void __launch_bounds__(EX_ROWS)
    k_assign_cuda_core(const T* __restrict__ X, const T* __restrict__ C,
                       const void* __restrict__ xn_in, const void* __restrict__ cn_in,
                       int64_t N, int64_t K, int64_t d, int32_t* __restrict__ idx_out,
                       void* __restrict__ mind_out, const int32_t* __restrict__ idx_prev,
                       int32_t* changed, const int32_t* __restrict__ list = nullptr,
                       const int32_t* __restrict__ list_cnt = nullptr) {
  using Acc = typename std::conditional<EXACT, double, float>::type;
  // Exact mode compares rounded T distances; low-precision mode compares fp32 scores.
  using Score = typename std::conditional<EXACT, T, float>::type;
  __shared__ T xs[EX_DC][EX_ROWS + 1];
  __shared__ T cs[EX_KT][EX_DC];
  __shared__ int32_t srow[LIST ? EX_ROWS : 1];
  const int64_t b = blockIdx.y;
  const int64_t row0 = (int64_t)blockIdx.x * EX_ROWS;
  const int tid = threadIdx.x;
  int64_t row = row0 + tid;
  if constexpr (LIST) {
    const int64_t cnt = list_cnt[b];
    if (row0 >= cnt) return;  // whole block: nothing listed here
    srow[tid] = row0 + tid < cnt ? list[b * N + row0 + tid] : -1;
    row = srow[tid] >= 0 ? srow[tid] : N;  // N = no row
    __syncthreads();
  }
  const T* Xb = X + b * N * d;
  const T* Cb = C + b * K * d;

  Score best = (Score)__int_as_float(0x7f800000);
  int32_t bi = -1;
  float xn_lp = 0.f;  // low-precision path: ||x||^2 accumulated on the fly
  Score xn_ex = (Score)0;
  if constexpr (EXACT) {
    if (row < N) xn_ex = reinterpret_cast<const T*>(xn_in)[b * N + row];
  }
  const float* cn_lp = reinterpret_cast<const float*>(cn_in);
  const T* cn_ex = reinterpret_cast<const T*>(cn_in);

  for (int64_t k0 = 0; k0 < K; k0 += EX_KT) {
    Acc acc[EX_KT];
#pragma unroll
    for (int kk = 0; kk < EX_KT; ++kk) acc[kk] = (Acc)0;
    for (int64_t j0 = 0; j0 < d; j0 += EX_DC) {
      __syncthreads();
      for (int e = tid; e < EX_ROWS * EX_DC; e += EX_ROWS) {
        int r = e / EX_DC, jj = e % EX_DC;
        int64_t gr = LIST ? (srow[r] >= 0 ? (int64_t)srow[r] : N) : row0 + r, gj = j0 + jj;
        xs[jj][r] = (gr < N && gj < d) ? Xb[gr * d + gj] : (T)0.f;
      }
      for (int e = tid; e < EX_KT * EX_DC; e += EX_ROWS) {
        int kk = e / EX_DC, jj = e % EX_DC;
        int64_t gk = k0 + kk, gj = j0 + jj;
        cs[kk][jj] = (gk < K && gj < d) ? Cb[gk * d + gj] : (T)0.f;
      }
      __syncthreads();
      const int jn = (int)((d - j0) < EX_DC ? (d - j0) : EX_DC);
      for (int jj = 0; jj < jn; ++jj) {
        const T xv = xs[jj][tid];
        if constexpr (!EXACT) {
          if (k0 == 0) {
            float f = to_f32(xv);
            xn_lp = fmaf(f, f, xn_lp);
          }
        }
#pragma unroll
        for (int kk = 0; kk < EX_KT; ++kk) {
          if constexpr (EXACT) {
            if constexpr (sizeof(T) == 4) {
              acc[kk] = __dadd_rn(acc[kk], (double)__fmul_rn(xv, cs[kk][jj]));
            } else {
              acc[kk] = __dadd_rn(acc[kk], __dmul_rn(xv, cs[kk][jj]));
            }
          } else {
            acc[kk] = fmaf(to_f32(xv), to_f32(cs[kk][jj]), acc[kk]);
          }
        }
      }
    }
#pragma unroll
    for (int kk = 0; kk < EX_KT; ++kk) {
      const int64_t k = k0 + kk;
      if (k < K) {
        Score v;
        if constexpr (EXACT) {
          T s;  // fl_T(xn + cn)
          if constexpr (sizeof(T) == 4) s = __fadd_rn(xn_ex, cn_ex[b * K + k]);
          else s = __dadd_rn(xn_ex, cn_ex[b * K + k]);
          double dv = __dsub_rn((double)s, __dmul_rn(2.0, acc[kk]));
          if (dv < 0.0) dv = 0.0;
          v = (T)dv;
        } else {
          v = fmaf(-2.f, acc[kk], cn_lp[b * K + k]);
        }
        if (v < best) {
          best = v;
          bi = (int32_t)k;
        }
      }
    }
  }
  bool ch = false;
  if (row < N) {
    const int64_t o = b * N + row;
    idx_out[o] = bi;
    if constexpr (EXACT) {
      reinterpret_cast<T*>(mind_out)[o] = best;
    } else {
      reinterpret_cast<float*>(mind_out)[o] = fmaxf(0.f, xn_lp + best);
    }
    if (idx_prev) ch = idx_prev[o] != bi;
  }
  if (changed && __any_sync(0xffffffffu, ch) && (tid & 31) == 0) atomicOr(changed, 1);
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_cn_pad(int dt, const void* C, int64_t B, int64_t K, int64_t d, int kpad,
                          float* cn_pad, cudaStream_t stream, float scale) {
  const int64_t n = B * kpad * 32;  // one warp per row
  const int th = 256;
  const unsigned grid = (unsigned)((n + th - 1) / th);
  if (dt == DT_BF16)
    k_cn_pad<__nv_bfloat16><<<grid, th, 0, stream>>>((const __nv_bfloat16*)C, B, K, d, kpad, cn_pad, scale);
  else if (dt == DT_F16)
    k_cn_pad<__half><<<grid, th, 0, stream>>>((const __half*)C, B, K, d, kpad, cn_pad, scale);
  else
    k_cn_pad<float><<<grid, th, 0, stream>>>((const float*)C, B, K, d, kpad, cn_pad, scale);
  return cudaGetLastError();
}

cudaError_t launch_row_norms_exact(int dt, const void* M, int64_t rows, int64_t d, void* out,
                                   cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  const int th = 128;
  const unsigned grid = (unsigned)((rows + th - 1) / th);
  if (rows >= 4096) {  // enough rows to fill the GPU with 128-row tiles
    if (dt == DT_F64)
      k_row_norms_staged<double><<<grid, th, 0, stream>>>((const double*)M, rows, d, (double*)out);
    else
      k_row_norms_staged<float><<<grid, th, 0, stream>>>((const float*)M, rows, d, (float*)out);
  } else if (dt == DT_F64) {
    k_row_norms_exact<double><<<grid, th, 0, stream>>>((const double*)M, rows, d, (double*)out);
  } else {
    k_row_norms_exact<float><<<grid, th, 0, stream>>>((const float*)M, rows, d, (float*)out);
  }
  return cudaGetLastError();
}

cudaError_t launch_assign_exact(int dt, const void* X, const void* C, const void* xn,
                                const void* cn, int64_t B, int64_t N, int64_t K, int64_t d,
                                int32_t* idx_out, void* mind_out, const int32_t* idx_prev,
                                int32_t* changed, cudaStream_t stream) {
  dim3 grid((unsigned)((N + EX_ROWS - 1) / EX_ROWS), (unsigned)B);
  if (dt == DT_F64)
    k_assign_cuda_core<double, true><<<grid, EX_ROWS, 0, stream>>>(
        (const double*)X, (const double*)C, xn, cn, N, K, d, idx_out, mind_out, idx_prev, changed);
  else
    k_assign_cuda_core<float, true><<<grid, EX_ROWS, 0, stream>>>(
        (const float*)X, (const float*)C, xn, cn, N, K, d, idx_out, mind_out, idx_prev, changed);
  return cudaGetLastError();
}

cudaError_t launch_assign_exact_rows(int dt, const void* X, const void* C, const void* xn,
                                     const void* cn, int64_t B, int64_t N, int64_t K, int64_t d,
                                     const int32_t* list, const int32_t* list_cnt,
                                     int32_t* idx_out, void* mind_out, const int32_t* idx_prev,
                                     int32_t* changed, cudaStream_t stream) {
  dim3 grid((unsigned)((N + EX_ROWS - 1) / EX_ROWS), (unsigned)B);
  if (dt == DT_F64)
    k_assign_cuda_core<double, true, true><<<grid, EX_ROWS, 0, stream>>>(
        (const double*)X, (const double*)C, xn, cn, N, K, d, idx_out, mind_out, idx_prev, changed,
        list, list_cnt);
  else
    k_assign_cuda_core<float, true, true><<<grid, EX_ROWS, 0, stream>>>(
        (const float*)X, (const float*)C, xn, cn, N, K, d, idx_out, mind_out, idx_prev, changed,
        list, list_cnt);
  return cudaGetLastError();
}

cudaError_t launch_assign_cuda_core_lowp(int dt, const void* X, const void* C, const float* cn,
                                         int64_t B, int64_t N, int64_t K, int64_t d,
                                         int32_t* idx_out, float* mind_out,
                                         const int32_t* idx_prev, int32_t* changed,
                                         cudaStream_t stream) {
  dim3 grid((unsigned)((N + EX_ROWS - 1) / EX_ROWS), (unsigned)B);
  // cn is the padded (B, kpad) vector; index it as (B, K) via a pitch of kpad
  // is not needed here: the caller passes a dense (B, K) view.
  if (dt == DT_BF16)
    k_assign_cuda_core<__nv_bfloat16, false><<<grid, EX_ROWS, 0, stream>>>(
        (const __nv_bfloat16*)X, (const __nv_bfloat16*)C, nullptr, cn, N, K, d, idx_out, mind_out,
        idx_prev, changed);
  else
    k_assign_cuda_core<__half, false><<<grid, EX_ROWS, 0, stream>>>(
        (const __half*)X, (const __half*)C, nullptr, cn, N, K, d, idx_out, mind_out, idx_prev,
        changed);
  return cudaGetLastError();
}

FK_MODULE_ANCHOR(assign_exact)

}  // namespace fk
