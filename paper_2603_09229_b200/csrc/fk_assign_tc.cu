// fk_assign_tc.cu -- FlashAssign on 5th-generation tensor cores (sm_100a).
//
// Replaces flash_assign (reference flash_assign.py:135-222, inner kernels
// _kernels.py:32-104) for bf16/fp16 data: the X.C^T contraction runs as a
// tcgen05.mma GEMM with operands staged by TMA and the fp32 accumulator in
// TMEM; the ||c||^2 bias and the online argmin are fused into the epilogue,
// so no N x K distance ever reaches HBM (the reference's zero-materialization
// property, flash_assign.py:1-15).
//
// Two kernels:
//  * fk_assign_tc2_kernel (default): persistent CTA pairs (cta_group::2, one
//    pair per TPC).  The leader issues M=256 N=256 K=16 MMAs into a double-
//    buffered TMEM accumulator; each CTA stages its 128 X rows (own producer
//    warp) and half of every C tile (C/bias producer warp).  The ||c||^2/2
//    bias rides in the GEMM as one extra K=16 step (A-negated main MMAs), so
//    the 8 epilogue warps only run a min tree per 32-column TMEM chunk.  See
//    the comments at tc2:: and DESIGN.md §4.
//  * fk_assign_tc_kernel (FK_ASSIGN_CTA=1, A/B only, d <= 128): the first
//    single-CTA design, kept for comparisons.  Warp 0 loads X / C / ||c||^2,
//    warp 1 issues M=128 N=256 MMAs, warps 4-11 run the epilogue with the
//    bias added per element (packed FFMA2 from smem).
// In both, a chunk's 32 scores are copied into a register-resident "winning
// chunk" only when some row of the warp improves, so the index is recovered
// once per row tile instead of being tracked per element.
// Tie rule (rowmin_merge, _kernels.py:64-82): strict < in ascending column
// order within a thread, first equal element within the winning chunk, and a
// lexicographic (value, index) merge across the two warpgroups -> the lowest
// centroid id among equal minima.
#include "fk_common.cuh"
#include "fk_kernels.h"
#include <cstdio>
#include <cstdlib>

// A/B build knobs: L2 policy of the X row-tile loads and the tensor maps' L2
// promotion (defaults are the measured choices)
#ifndef FK_X_HINT
#define FK_X_HINT kEvictFirst
#endif
#ifndef FK_TMAP_PROMO
#define FK_TMAP_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif

namespace fk {

namespace tc {
constexpr int BM = 128;                  // rows per tile = TMEM lanes
constexpr int BN = 256;                  // centroids per column tile
constexpr int STAGES = 4;                // C ring depth (32 KB each)
constexpr int KATOMS_MAX = 2;            // d <= 128 (64 bf16 = 128 B per atom)
constexpr int A_ATOM = BM * 128;         // 16 KB
constexpr int A_SLOT = KATOMS_MAX * A_ATOM;
constexpr int B_STAGE = BN * 128;        // 32 KB
constexpr int CN_SLOTS = 4;              // ||c||^2 ring (1 KB per column tile)
constexpr int OFF_A = 0;
constexpr int OFF_B = OFF_A + 2 * A_SLOT;            // 64 KB
constexpr int OFF_CN = OFF_B + STAGES * B_STAGE;     // 192 KB
constexpr int OFF_XCH = OFF_CN + CN_SLOTS * BN * 4;  // 196 KB
constexpr int OFF_BAR = OFF_XCH + BM * 8;
constexpr int NBARS = 16 + 2 * CN_SLOTS;
constexpr int SMEM_USED = OFF_BAR + NBARS * 8 + 16;
constexpr int SMEM_BYTES = SMEM_USED + 1024;         // alignment slack
constexpr int THREADS = 384;
static_assert(SMEM_BYTES <= 232448, "exceeds 227 KB dynamic shared memory");
}  // namespace tc

struct TcArgs {
  int B, N, K, d;
  int katoms;           // ceil(d / 64): 1 or 2 (single-CTA kernel), 1..4 (pair kernel)
  int tiles_per_batch;  // ceil(N / 128)
  int total_tiles;      // B * tiles_per_batch
  int ncol;             // ceil(K / 256)
  int kpad;             // ncol * 256
  const float* cn;      // (B, kpad) ||c||^2, +inf beyond K
  int32_t* idx_out;     // (B, N)
  float* mind_out;      // (B, N)
  const int32_t* idx_prev;
  int32_t* changed;
  int debug_mode;  // 0 normal; 1 epilogue skips math (MMA/TMA bound); 2 MMA skipped (epilogue bound)
  int epi2;        // 1: bias-in-GEMM epilogue processes 32-column chunks in pairs
  unsigned long long* trace;  // debug timeline (FK_ASSIGN_TRACE), nullptr normally
  // split (f32/f64 data, fk_assign_split.cu): X and C are bf16 [hi | lo] rows
  // of 2*ns K=16 steps; the MMA runs hi.hi + hi.lo + lo.hi per step and the
  // epilogue also reports a lower bound on each row's second-best score.
  int ns;
  float* second_out;  // (B, N) second-best score bound (split only)
  // split: the epilogue's own certificate (margin from an upper bound of |x|
  // read off the [hi | lo] tile and cmax) and, for rows it cannot certify,
  // the column bases of every 32-column chunk whose minimum came within the
  // margin of the running best (the only places the exact argmin can be)
  const unsigned int* cmax;  // (B) float bits, upper bound of max_k |c_k|
  int8_t* stat_out;          // (B, N) 0 certified, 1 candidate chunks listed, 2 full fallback
  int32_t* cand_rec;         // records [row, n, chunk bases...], FK_SPLIT_REC ints each
  int32_t* cand_cnt;         // record count (device)
  int cand_cap;
  // the update's block histograms, folded into the epilogue (fk_assign_hist):
  // row i of batch element b adds 1 to hist_tab[(b * hist_bpb + i / hist_per) * K + id]
  // (an id outside [0, K) to hist_inval[b * hist_bpb + i / hist_per]) -- the
  // table k_hist would have built; nullptr: off
  int32_t* hist_tab;
  int32_t* hist_inval;
  int hist_bpb, hist_per;
  // (B, N) fp32 ||x||^2 precomputed by k_row_norms_tc with the epilogue's own
  // arithmetic (X is fixed through a Lloyd run): loaded instead of summing the
  // row from the shared-memory tile every row tile; nullptr: summed here
  const float* xn_in;
  // first row tile of this launch (the pair kernel beside the multicast quads
  // takes the tiles after theirs); 0 otherwise
  int tile0;
};

constexpr int SPLIT_NREC = 4;                  // near chunks kept per thread (per column half)
constexpr int FK_SPLIT_REC = 2 + 2 * SPLIT_NREC;
static_assert(FK_SPLIT_REC == kSplitRecInts, "candidate record layout (fk_kernels.h)");

// Debug timeline: events of pair 0 / tile window [TR_G0, TR_G0 + TR_N) only.
constexpr int TR_N = 32, TR_EV = 8;
#ifdef FK_ASSIGN_TRACE_BUILD
constexpr int TR_G0 = 16;
#endif
// Bound-analysis modes (FK_ASSIGN_DEBUG_MODE) exist only in debug builds
// (FK_BUILD_DEBUG=1 -> -DFK_ASSIGN_DEBUG_BUILD); elsewhere the mode is the
// constant 0 and every check folds away.
#ifdef FK_ASSIGN_DEBUG_BUILD
FK_DEV int dbg_mode(const TcArgs& p) { return p.debug_mode; }
#else
FK_DEV constexpr int dbg_mode(const TcArgs&) { return 0; }
#endif

// Compiled in only for timeline builds (FK_BUILD_TRACE=1 -> -DFK_ASSIGN_TRACE_BUILD):
// the role warps share their SM sub-partitions with ALU-bound epilogue warps,
// so every instruction on the MMA warp's per-tile path costs issue slots it
// waits for (the checks alone were ~20 instructions per tile).
#ifdef FK_ASSIGN_TRACE_BUILD
FK_DEV void trace_ev(const TcArgs& p, uint32_t g, int ev) {
  if (p.trace && g >= TR_G0 && g < TR_G0 + TR_N) p.trace[(g - TR_G0) * TR_EV + ev] = clock64();
}
#else
FK_DEV void trace_ev(const TcArgs&, uint32_t, int) {}
#endif

// ||x||^2 of one row of the staged X tile over the 16-byte chunk positions
// [j0, j1) of every K atom (the caller may split the 8 positions between
// warpgroups; any split covers each element exactly once).
template <int FMT>
FK_DEV float row_norm_smem(const uint8_t* a_slot, int row, int katoms, int lane, int j0 = 0,
                           int j1 = 8) {
  float acc = 0.f;
  for (int ka = 0; ka < katoms; ++ka) {
    const uint4* r = reinterpret_cast<const uint4*>(a_slot + ka * tc::A_ATOM + row * 128);
#pragma unroll
    for (int j = j0; j < j1; ++j) {
      uint4 w = r[(j + lane) & 7];
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float lo, hi;
        if (FMT == 1) {
          lo = __uint_as_float(ws[e] << 16);
          hi = __uint_as_float(ws[e] & 0xffff0000u);
        } else {
          __half2 h = *reinterpret_cast<__half2*>(&ws[e]);
          float2 f = __half22float2(h);
          lo = f.x;
          hi = f.y;
        }
        acc = fmaf(lo, lo, acc);
        acc = fmaf(hi, hi, acc);
      }
    }
  }
  return acc;
}

// One 32-column chunk: bias, chunk minimum, conditional capture of the
// winning chunk's scores (registers; only when some row of the warp improves).
FK_DEV void epi_chunk(uint32_t (&v)[32], uint32_t cn_addr, int colbase, float& M, int& best,
                      float (&bestv)[32]) {
  const float2 m2 = make_float2(-2.f, -2.f);
  float* s = reinterpret_cast<float*>(v);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 cc = lds128(cn_addr + 16 * j);
    float2 r0 = ffma2(make_float2(s[4 * j], s[4 * j + 1]), m2, make_float2(cc.x, cc.y));
    float2 r1 = ffma2(make_float2(s[4 * j + 2], s[4 * j + 3]), m2, make_float2(cc.z, cc.w));
    s[4 * j] = r0.x;
    s[4 * j + 1] = r0.y;
    s[4 * j + 2] = r1.x;
    s[4 * j + 3] = r1.y;
  }
  float a[11];
#pragma unroll
  for (int j = 0; j < 10; ++j) a[j] = fmin3(s[3 * j], s[3 * j + 1], s[3 * j + 2]);
  a[10] = fminf(s[30], s[31]);
  const float b0 = fmin3(a[0], a[1], a[2]);
  const float b1 = fmin3(a[3], a[4], a[5]);
  const float b2 = fmin3(a[6], a[7], a[8]);
  const float b3 = fminf(a[9], a[10]);
  const float mc = fmin3(b0, b1, fminf(b2, b3));
  const bool p = mc < M;
  if (__any_sync(0xffffffffu, p)) {
#pragma unroll
    for (int j = 0; j < 32; ++j) bestv[j] = p ? s[j] : bestv[j];
  }
  M = p ? mc : M;
  best = p ? colbase : best;
}

template <int FMT>
__global__ void __launch_bounds__(tc::THREADS, 1)
    fk_assign_tc_kernel(const __grid_constant__ CUtensorMap tmx,
                        const __grid_constant__ CUtensorMap tmc, const TcArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem + tc::OFF_A;
  uint8_t* sB = smem + tc::OFF_B;
  float* sCN = reinterpret_cast<float*>(smem + tc::OFF_CN);
  float* xch_m = reinterpret_cast<float*>(smem + tc::OFF_XCH);
  int* xch_i = reinterpret_cast<int*>(smem + tc::OFF_XCH + tc::BM * 4);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + tc::OFF_BAR);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 2;
  uint64_t* b_full = bars + 4;
  uint64_t* b_empty = bars + 8;
  uint64_t* t_full = bars + 12;
  uint64_t* t_empty = bars + 14;
  uint64_t* cn_full = bars + 16;
  uint64_t* cn_empty = bars + 16 + tc::CN_SLOTS;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + tc::NBARS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmx);
    tma_prefetch_desc(&tmc);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_empty[s], 1 + 4);  // MMA commit + 4 warps of epilogue WG0 (row norms)
      mbar_init(&t_full[s], 1);
      mbar_init(&t_empty[s], 8);      // every epilogue warp
    }
    for (int s = 0; s < tc::STAGES; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    for (int s = 0; s < tc::CN_SLOTS; ++s) {
      mbar_init(&cn_full[s], 1);
      mbar_init(&cn_empty[s], 8);  // every epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t stage = 0, sphase = 0;
      const uint32_t a_bytes = p.katoms * tc::A_ATOM;
      auto load_a = [&](int t, int j) {
        const int slot = j & 1;
        const int b = t / p.tiles_per_batch;
        const int row0 = (t - b * p.tiles_per_batch) * tc::BM;
        mbar_wait(&a_empty[slot], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&a_full[slot], a_bytes);
        for (int ka = 0; ka < p.katoms; ++ka)
          tma_load_3d(sA + slot * tc::A_SLOT + ka * tc::A_ATOM, &tmx, &a_full[slot], ka * 64, row0,
                      b, kEvictFirst);
      };
      int i = 0;
      uint32_t g = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++i) {
        const int b = t / p.tiles_per_batch;
        if (i == 0) load_a(t, 0);
        for (int c = 0; c < p.ncol; ++c, ++g) {
          {  // ||c||^2 slice of this column tile
            const uint32_t slot = g % tc::CN_SLOTS;
            mbar_wait(&cn_empty[slot], ((g / tc::CN_SLOTS) & 1) ^ 1);
            mbar_arrive_expect_tx(&cn_full[slot], tc::BN * 4);
            bulk_load(sCN + slot * tc::BN, p.cn + (size_t)b * p.kpad + (size_t)c * tc::BN,
                      tc::BN * 4, &cn_full[slot]);
          }
          for (int ka = 0; ka < p.katoms; ++ka) {
            mbar_wait(&b_empty[stage], sphase ^ 1);
            mbar_arrive_expect_tx(&b_full[stage], tc::B_STAGE);
            tma_load_3d(sB + stage * tc::B_STAGE, &tmc, &b_full[stage], ka * 64, c * tc::BN, b,
                        kEvictLast);
            if (++stage == tc::STAGES) {
              stage = 0;
              sphase ^= 1;
            }
          }
          if (c == 0) {
            const int t2 = t + gridDim.x;
            if (t2 < p.total_tiles) load_a(t2, i + 1);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issue
    if (lane == 0) {
      const uint32_t idesc = make_idesc_f16(FMT, tc::BM, tc::BN);
      uint32_t stage = 0, sphase = 0, g = 0;
      int i = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++i) {
        const int slot = i & 1;
        mbar_wait(&a_full[slot], (i >> 1) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sA + slot * tc::A_SLOT);
        for (int c = 0; c < p.ncol; ++c, ++g) {
          const uint32_t buf = g & 1;
          mbar_wait(&t_empty[buf], ((g >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + buf * tc::BN;
          for (int ka = 0; ka < p.katoms; ++ka) {
            mbar_wait(&b_full[stage], sphase);
            tc_fence_after();
            const uint32_t aa = a_base + ka * tc::A_ATOM;
            const uint32_t bb = smem_u32(sB + stage * tc::B_STAGE);
            if (dbg_mode(p) != 2) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc_mma_f16(d_tmem, make_sdesc_sw128(aa + k * 32), make_sdesc_sw128(bb + k * 32),
                           idesc, (ka | k) != 0);
            }
            tc_commit(&b_empty[stage]);
            if (++stage == tc::STAGES) {
              stage = 0;
              sphase ^= 1;
            }
          }
          tc_commit(&t_full[buf]);
        }
        tc_commit(&a_empty[slot]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    const int wg = ew >> 2;         // column half of every tile
    const int q = warp & 3;         // TMEM lane quarter
    const int row = q * 32 + lane;  // tile row owned by this thread
    uint32_t g = 0;
    int i = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++i) {
      const int b = t / p.tiles_per_batch;
      const int row0 = (t - b * p.tiles_per_batch) * tc::BM;
      const int slot = i & 1;
      float M = __int_as_float(0x7f800000);
      int best = -1;
      float bestv[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) bestv[j] = M;
      float xn = 0.f;
      for (int c = 0; c < p.ncol; ++c, ++g) {
        const uint32_t buf = g & 1;
        const uint32_t cslot = g % tc::CN_SLOTS;
        mbar_wait(&t_full[buf], (g >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + buf * tc::BN + wg * 128;
        uint32_t va[32], vb[32];
        FK_TMEM_LD_32x32b_X32(taddr, va);
        if (c == 0 && wg == 0) {
          xn = row_norm_smem<FMT>(sA + slot * tc::A_SLOT, row, p.katoms, lane);
          __syncwarp();
          if (lane == 0) mbar_arrive(&a_empty[slot]);
        }
        mbar_wait(&cn_full[cslot], (g / tc::CN_SLOTS) & 1);
        const uint32_t cnp = smem_u32(sCN + cslot * tc::BN + wg * 128);
        const int col0 = c * tc::BN + wg * 128;
        if (dbg_mode(p) == 1) {
          FK_TMEM_WAIT_LD(va);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&t_empty[buf]);
            mbar_arrive(&cn_empty[cslot]);
          }
          M = fminf(M, __uint_as_float(va[0]));
          continue;
        }
        FK_TMEM_WAIT_LD(va);
        FK_TMEM_LD_32x32b_X32(taddr + 32, vb);
        epi_chunk(va, cnp, col0, M, best, bestv);
        FK_TMEM_WAIT_LD(vb);
        FK_TMEM_LD_32x32b_X32(taddr + 64, va);
        epi_chunk(vb, cnp + 128, col0 + 32, M, best, bestv);
        FK_TMEM_WAIT_LD(va);
        FK_TMEM_LD_32x32b_X32(taddr + 96, vb);
        epi_chunk(va, cnp + 256, col0 + 64, M, best, bestv);
        FK_TMEM_WAIT_LD(vb);
        // every TMEM read of this buffer has landed: hand it back to the MMA warp
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[buf]);
        epi_chunk(vb, cnp + 384, col0 + 96, M, best, bestv);
        __syncwarp();
        if (lane == 0) mbar_arrive(&cn_empty[cslot]);
      }
      // recover the index inside the winning chunk (first equal element)
      int idx = -1;
      if (best >= 0) {
        int found = 31;
#pragma unroll
        for (int j = 31; j >= 0; --j) found = (bestv[j] == M) ? j : found;
        idx = best + found;
      }
      if (wg == 1) {
        xch_m[row] = M;
        xch_i[row] = idx;
      }
      named_bar_sync(1, 256);
      if (wg == 0) {
        const float M1 = xch_m[row];
        const int i1 = xch_i[row];
        if (M1 < M || (M1 == M && i1 >= 0 && (idx < 0 || i1 < idx))) {
          M = M1;
          idx = i1;
        }
        const int grow = row0 + row;
        bool ch = false;
        if (grow < p.N) {
          const size_t o = (size_t)b * p.N + grow;
          p.idx_out[o] = idx;
          p.mind_out[o] = fmaxf(0.f, xn + M);
          if (p.idx_prev) ch = p.idx_prev[o] != idx;
        }
        if (p.changed && __any_sync(0xffffffffu, ch) && lane == 0) atomicOr(p.changed, 1);
      }
      named_bar_sync(2, 256);
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

// ====================================================================
// CTA-pair variant (cta_group::2): the two CTAs of a cluster own 128 rows
// each and compute a 256 x 256 tile with one MMA stream issued by the leader
// CTA.  Each CTA stages only HALF of every C tile (128 centroids), so the
// L2 -> SM traffic and the shared-memory footprint of C halve; the per-SM
// epilogue work is unchanged.
// ====================================================================
namespace tc2 {
constexpr int BM = 128;                  // rows per CTA (TMEM lanes)
constexpr int BN = 256;                  // centroids per pair tile
constexpr int BNH = 128;                 // centroids staged per CTA
constexpr int NBUF = 2;                  // TMEM accumulators (2 x 256 columns)
constexpr int A_ATOM = BM * 128;         // 16 KB
constexpr int B_STAGE = BNH * 128;       // 16 KB per CTA
constexpr int STAGES = 6;
constexpr int CN_SLOTS = 6;              // ||c||^2 ring (bias in the epilogue)
constexpr int EXT_ROW = 32;              // 16 bf16: [hi, mid, lo, 0...] of ||c||^2 / 2
constexpr int EXT_SLOT = BNH * EXT_ROW;  // 4 KB per CTA per column tile
constexpr int EXT_SLOTS = 4;             // bias-in-GEMM operand ring
// Layout: the small rings first, then ONE operand region shared by the X
// row-tile ring and the C stage ring, sized per d (see operand_plan).
constexpr int OFF_AEXT = 0;                                // constant ones operand (4 KB)
constexpr int OFF_EXT = OFF_AEXT + BM * EXT_ROW;
constexpr int OFF_CN = OFF_EXT + EXT_SLOTS * EXT_SLOT;
constexpr int OFF_XCH = OFF_CN + CN_SLOTS * BN * 4;
constexpr int OFF_BAR = OFF_XCH + BM * 48;  // [min | idx | ||x||^2 part | second | 8 near-chunk words]
constexpr int A_SLOTS_MAX = 8;
constexpr int NBARS = 2 * A_SLOTS_MAX + 2 * NBUF + 2 * STAGES + 2 * CN_SLOTS + 2 * EXT_SLOTS;
constexpr int OFF_OPS = ((OFF_BAR + NBARS * 8 + 16) + 1023) & ~1023;  // 1 KB aligned (SW128)
constexpr int SMEM_BYTES = 232448;                          // 227 KB: the whole opt-in carve-out
constexpr int OPS_BYTES = SMEM_BYTES - 1024 - OFF_OPS;      // minus the base-alignment slack
constexpr int THREADS = 384;
constexpr int KATOMS_MAX = 4;                               // d <= 256
static_assert(2 * KATOMS_MAX * A_ATOM + 4 * B_STAGE <= OPS_BYTES, "d = 256 plan does not fit");
static_assert(2 * 2 * A_ATOM + STAGES * B_STAGE <= OPS_BYTES, "d = 128 plan does not fit");
static_assert(8 * A_ATOM + 4 * B_STAGE <= OPS_BYTES, "d = 64 plan does not fit");
// (X slots, C stages) per K-atom count: deep X prefetch for short rows,
// deep C prefetch otherwise, at least one column tile of C for d = 256.
__host__ __device__ inline void operand_plan(int katoms, int& a_slots, int& b_stages) {
  if (katoms == 1) {
    a_slots = 8;  // 8 x 16 KB: X prefetch deep enough for short row tiles (config 4)
    b_stages = 4;
  } else if (katoms == 4) {
    a_slots = 2;
    b_stages = 4;
  } else {
    a_slots = 2;
    b_stages = STAGES;
  }
}
}  // namespace tc2

// Epilogue chunk when the bias is already in the accumulator (s = ||c||^2/2 - x.c).
template <bool S = false>
FK_DEV void epi_chunk_aug(uint32_t (&v)[32], int colbase, float& M, int& best, float (&bestv)[32],
                          float& m2, float& mc_out) {
  const float* s = reinterpret_cast<const float*>(v);
  float a[11];
#pragma unroll
  for (int j = 0; j < 10; ++j) a[j] = fmin3(s[3 * j], s[3 * j + 1], s[3 * j + 2]);
  a[10] = fminf(s[30], s[31]);
  const float b0 = fmin3(a[0], a[1], a[2]);
  const float b1 = fmin3(a[3], a[4], a[5]);
  const float b2 = fmin3(a[6], a[7], a[8]);
  const float b3 = fminf(a[9], a[10]);
  const float mc = fmin3(b0, b1, fminf(b2, b3));
  const bool p = mc < M;
  // split: every chunk other than the winner's bounds the second best from
  // below by its minimum (the winner's own chunk is scanned at the end)
  if constexpr (S) {
    m2 = fminf(m2, fmaxf(M, mc));
    mc_out = mc;
  }
  if (__any_sync(0xffffffffu, p)) {
#pragma unroll
    for (int j = 0; j < 32; ++j) bestv[j] = p ? s[j] : bestv[j];
  }
  M = p ? mc : M;
  best = p ? colbase : best;
}

FK_DEV float min_tree32(const float* s) {
  float a[11];
#pragma unroll
  for (int j = 0; j < 10; ++j) a[j] = fmin3(s[3 * j], s[3 * j + 1], s[3 * j + 2]);
  a[10] = fminf(s[30], s[31]);
  const float b0 = fmin3(a[0], a[1], a[2]);
  const float b1 = fmin3(a[3], a[4], a[5]);
  const float b2 = fmin3(a[6], a[7], a[8]);
  const float b3 = fminf(a[9], a[10]);
  return fmin3(b0, b1, fminf(b2, b3));
}

// Two adjacent chunks at once: independent min trees (ILP), one warp vote and
// one conditional copy per pair.  Chunk a holds the lower columns, so strict
// '<' in order a then b keeps the lowest index on ties, as epi_chunk_aug does.
template <bool S = false>
FK_DEV void epi_chunk2_aug(const uint32_t (&va)[32], const uint32_t (&vb)[32], int cola, int colb,
                           float& M, int& best, float (&bestv)[32], float& m2, float& mca_out,
                           float& mcb_out) {
  const float* sa = reinterpret_cast<const float*>(va);
  const float* sb = reinterpret_cast<const float*>(vb);
  const float mca = min_tree32(sa);
  const float mcb = min_tree32(sb);
  const bool pa = mca < M;
  const float Ma = pa ? mca : M;
  const bool pb = mcb < Ma;
  if constexpr (S) {
    m2 = fminf(fminf(m2, fmaxf(M, mca)), fmaxf(Ma, mcb));
    mca_out = mca;
    mcb_out = mcb;
  }
  if (__any_sync(0xffffffffu, pa || pb)) {
#pragma unroll
    for (int j = 0; j < 32; ++j) bestv[j] = pb ? sb[j] : (pa ? sa[j] : bestv[j]);
  }
  M = pb ? mcb : Ma;
  best = pb ? colb : (pa ? cola : best);
}

// Split tile row: upper bound of |x| from the [hi | lo] bf16 operand row,
// |x| <= |hi| + |lo| + 2^-16 |x| (hi columns: the first 16 ns of the row).
// Physical 16-byte chunk p of a 128-byte-swizzled row r holds logical chunk
// p ^ (r & 7).
FK_DEV float split_norm_ub(const uint8_t* a_slot, int row, int katoms, int ns, int lane) {
  float sh = 0.f, sl = 0.f;
  for (int ka = 0; ka < katoms; ++ka) {
    const uint4* r = reinterpret_cast<const uint4*>(a_slot + ka * tc::A_ATOM + row * 128);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int pc = (j + lane) & 7;
      const bool hi = ka * 64 + 8 * (pc ^ (row & 7)) < 16 * ns;
      uint4 w = r[pc];
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float lo = __uint_as_float(ws[e] << 16), hv = __uint_as_float(ws[e] & 0xffff0000u);
        acc = fmaf(lo, lo, acc);
        acc = fmaf(hv, hv, acc);
      }
      if (hi) sh += acc;
      else sl += acc;
    }
  }
  return (sqrtf(sh) + sqrtf(sl)) * (1.0f + 0x1p-10f) + 0x1p-60f;
}

// BIAS = 1 (bias-in-GEMM): the ||c||^2 bias rides in the GEMM as one extra
//              K=16 step (A_ext = ones, B_ext = 3-way bf16 split of
//              ||c||^2/2, main MMAs negate A), so the epilogue is a pure
//              min-reduction.
// BIAS = 2 (TMEM seed): after draining a TMEM accumulator the epilogue warps
//              store ||c||^2/2 of the tile that will reuse it (two tiles
//              ahead) into it with tcgen05.st; the MMAs (A negated)
//              accumulate onto the seed.  No extra MMA step, no fp16 range
//              issue, still a pure min-reduction epilogue.
// BIAS = 0 (epilogue bias): bias added in the epilogue from a smem ring.
// MC (fk_assign_tc2q_kernel): a cluster of two CTA pairs that take the two
//              row tiles of a tile pair in lockstep and share every C tile:
//              each CTA loads half of its half-tile and multicasts it to the
//              CTA of the same pair rank in the other pair, so C crosses L2
//              once per two row tiles (B = 1, bias in the GEMM, K > 256).
template <int FMT, int BIAS, bool ALT, bool SPLIT, bool MC>
FK_DEV void assign_tc2_body(const CUtensorMap& tmx, const CUtensorMap& tmc,
                            const CUtensorMap& tmext, const TcArgs& p) {
  using namespace tc2;
  static_assert(!MC || (BIAS == 1 && !ALT && !SPLIT), "multicast pairs: bias in the GEMM only");
  constexpr bool AUG = BIAS == 1;   // bias as an extra MMA step
  constexpr bool SEED = BIAS == 2;  // bias seeded into TMEM by the epilogue
  constexpr bool EPI = BIAS == 0;   // bias added in the epilogue
  constexpr bool NEG = BIAS != 0;   // accumulator holds ||c||^2/2 - x.c
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem + OFF_OPS;
  uint8_t* sB;
  uint8_t* sAext = smem + OFF_AEXT;
  uint8_t* sExt = smem + OFF_EXT;
  float* sCN = reinterpret_cast<float*>(smem + OFF_CN);
  float* xch_m = reinterpret_cast<float*>(smem + OFF_XCH);
  int* xch_i = reinterpret_cast<int*>(smem + OFF_XCH + BM * 4);
  float* xch_xn = reinterpret_cast<float*>(smem + OFF_XCH + BM * 8);
  float* xch_m2 = reinterpret_cast<float*>(smem + OFF_XCH + BM * 12);
  int32_t* xch_rec = reinterpret_cast<int32_t*>(smem + OFF_XCH + BM * 16);  // [row][8]: n, bases
  static_assert(!SPLIT || BIAS == 1, "split runs with the bias in the GEMM");
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + A_SLOTS_MAX;
  uint64_t* t_full = bars + 2 * A_SLOTS_MAX;
  uint64_t* t_empty = t_full + NBUF;
  uint64_t* b_full = t_empty + NBUF;
  uint64_t* b_empty = b_full + STAGES;
  uint64_t* cn_full = b_empty + STAGES;
  uint64_t* cn_empty = cn_full + CN_SLOTS;
  uint64_t* ext_full = cn_empty + CN_SLOTS;
  uint64_t* ext_empty = ext_full + EXT_SLOTS;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + NBARS);

  // Warp roles.  The SMSP arbiter favours the highest eligible warp id, so the
  // latency-critical single-thread roles sit above the eight epilogue warps
  // (0-7): 8 = C / bias producer, 9 = MMA issuer (leader CTA), 10 = TMEM
  // allocator, 11 = ones-operand init, then the X row-tile producer.
  constexpr int W_PRODUCER = 8, W_MMA = 9, W_TMEM = 10, W_INIT = 11;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = MC ? (crank & 1u) : crank;  // rank within the pair
  const uint32_t lead = MC ? (crank & 2u) : 0u;     // cluster rank of the pair's leader
  const uint16_t pmask = (uint16_t)(0x3u << lead);  // this pair's two CTAs
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  // row tiles of this pair: t_first, t_first + t_step, ... < t_end.  MC: the
  // quad's pairs take tiles 2v and 2v + 1 of the same tile pair v, so t_end is
  // rounded up to even and a pair may run one dummy tile (loads the last real
  // tile, writes nothing) to keep the shared C stream in step.
  const int t_first = MC ? 2 * (int)(blockIdx.x >> 2) + (int)(crank >> 1) : pair;
  const int t_step = MC ? 2 * (int)(gridDim.x >> 2) : npairs;
  const int t_end = MC ? ((p.total_tiles + 1) & ~1) : p.total_tiles;
  // X row-tile ring: the 64 KB A region holds 2 slots of 2 K-atoms (d <= 128)
  // or 4 slots of 1 atom (d <= 64): deeper prefetch when a row tile is short.
  // X row-tile ring + C stage ring share the 160 KB operand region: d <= 64
  // (one K-atom per tile) takes 6 X slots + 4 C stages -- short row tiles need
  // the deeper X prefetch -- d <= 128 takes 2 X slots + 6 C stages.
  int a_slots, b_stages;
  operand_plan(p.katoms, a_slots, b_stages);
  const int a_slot_bytes = p.katoms * A_ATOM;
  sB = sA + a_slots * a_slot_bytes;
  // ALT (single-column-tile rows, K <= 256): the two epilogue warpgroups take
  // alternate tiles (whole rows each, two tiles in flight, no merge) instead
  // of splitting every tile's columns.
  constexpr bool alt = ALT;
  const int epi_warps_per_buf = alt ? 4 : 8;

  if (warp == W_PRODUCER && lane == 0) {
    tma_prefetch_desc(&tmx);
    tma_prefetch_desc(&tmc);
    if (AUG) tma_prefetch_desc(&tmext);
    for (int s = 0; s < A_SLOTS_MAX; ++s) {
      mbar_init(&a_full[s], 1);       // leader's expect_tx (both CTAs' bytes)
      // pair-MMA commit + the row-norm warps (none with precomputed norms: the
      // slot is free as soon as the MMA has read it)
      mbar_init(&a_empty[s], 1 + ((!SPLIT && p.xn_in) ? 0 : (ALT ? 4 : 8)));
    }
    for (int s = 0; s < NBUF; ++s) {
      mbar_init(&t_full[s], 1);
      mbar_init(&t_empty[s], 2 * epi_warps_per_buf);  // epilogue warps of both CTAs
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], MC ? 2 : 1);  // MC: both pairs' MMAs read the stage
    }
    for (int s = 0; s < CN_SLOTS; ++s) {
      mbar_init(&cn_full[s], 1);
      mbar_init(&cn_empty[s], epi_warps_per_buf);
    }
    for (int s = 0; s < EXT_SLOTS; ++s) {
      mbar_init(&ext_full[s], 1);
      mbar_init(&ext_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (AUG && warp == W_INIT) {
    // A_ext rows = [1,1,1,0,0,0,0,0] in BOTH 16-byte halves: invariant under
    // the 32-byte swizzle, and only columns 0-2 of B_ext are non-zero.
    const uint32_t one = 0x3F80u;  // bf16 1.0 (bias MMA is bf16 x bf16 for any data type)
    const uint4 v = make_uint4(one | (one << 16), one, 0u, 0u);
    uint4* dst = reinterpret_cast<uint4*>(sAext);
    for (int i = lane; i < BM * 2; i += 32) dst[i] = v;
    fence_proxy_async_smem();
  }
  if (warp == W_TMEM) tmem_alloc_cg2<512>(tmem_holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == W_PRODUCER) {
    // ------------------------------------------------------------ producer (both CTAs)
    // C tiles (+ bias operand / ||c||^2 ring); X row tiles come from their own
    // warp below, so waiting for a free X slot never stalls the C prefetch.
    // The whole warp runs the loop (barrier and index arithmetic on the uniform
    // datapath, which the ALU-bound epilogue warps of this sub-partition do not
    // contend for); one elected lane issues each copy.
    {
      uint32_t stage = 0, sphase = 0;
      uint32_t g = 0;
      for (int t = t_first; t < t_end; t += t_step) {
        const int b = MC ? 0 : (p.tile0 + t) / p.tiles_per_batch;
        for (int c = 0; c < p.ncol; ++c, ++g) {
          // debug mode 4 (bound analysis, wrong results): C and bias operands
          // loaded once per ring slot, then reused as they are
          // (5: the bias operand only, 6: C only)
          const bool warm4 = g >= (uint32_t)(EXT_SLOTS + b_stages);
          const bool skip4 = warm4 && (dbg_mode(p) == 4 || dbg_mode(p) == 6);
          const bool skipx = warm4 && (dbg_mode(p) == 4 || dbg_mode(p) == 5);
          if (AUG) {
            const uint32_t slot = g % EXT_SLOTS;
            mbar_wait(&ext_empty[slot], ((g / EXT_SLOTS) & 1) ^ 1);
            if (elect_one()) {
              if (skipx) {
                if (leader) mbar_arrive(&ext_full[slot]);
              } else {
                if (leader) mbar_arrive_expect_tx(&ext_full[slot], 2 * EXT_SLOT);
                tma_load_3d_cg2(sExt + slot * EXT_SLOT, &tmext, mapa_shared(smem_u32(&ext_full[slot]), lead),
                                0, c * BN + rank * BNH, b, kEvictLast);
              }
            }
            __syncwarp();
          } else {
            const uint32_t slot = g % CN_SLOTS;
            mbar_wait(&cn_empty[slot], ((g / CN_SLOTS) & 1) ^ 1);
            if (elect_one()) {
              mbar_arrive_expect_tx(&cn_full[slot], BN * 4);
              bulk_load(sCN + slot * BN, p.cn + (size_t)b * p.kpad + (size_t)c * BN, BN * 4,
                        &cn_full[slot]);
            }
            __syncwarp();
          }
          for (int ka = 0; ka < p.katoms; ++ka) {
            mbar_wait(&b_empty[stage], sphase ^ 1);
            if (elect_one()) {
              if (skip4) {
                if (leader) mbar_arrive(&b_full[stage]);
              } else {
                if (leader) mbar_arrive_expect_tx(&b_full[stage], 2 * B_STAGE);
                if constexpr (MC) {  // half of the half-tile, to this CTA and its twin
                  const uint32_t pq = crank >> 1;
                  tma_load_3d_cg2_mc(sB + stage * B_STAGE + pq * (B_STAGE / 2), &tmc,
                                     mapa_shared(smem_u32(&b_full[stage]), lead),
                                     (uint16_t)(0x5u << rank), ka * 64,
                                     c * BN + rank * BNH + pq * (BNH / 2), b, kEvictLast);
                } else {
                  tma_load_3d_cg2(sB + stage * B_STAGE, &tmc, mapa_shared(smem_u32(&b_full[stage]), 0),
                                  ka * 64, c * BN + rank * BNH, b, kEvictLast);
                }
              }
            }
            __syncwarp();
            if (++stage == b_stages) {
              stage = 0;
              sphase ^= 1;
            }
          }
          if (pair == 0 && leader && lane == 0 && dbg_mode(p) != 3) trace_ev(p, g, 5);
        }
      }
    }
  } else if (warp == W_INIT) {
    // ------------------------------------------------------------ X row-tile producer (both CTAs)
    // (warp-wide loop, elected issue: as the C producer above)
    {
      const uint32_t a_bytes = p.katoms * A_ATOM;
      int j = 0, aslot = 0;
      uint32_t aphase = 0;
      for (int t = t_first; t < t_end; t += t_step, ++j) {
        const int slot = aslot;  // j % a_slots, without a division per tile
        const uint32_t aph = aphase;
        if (++aslot == a_slots) {
          aslot = 0;
          aphase ^= 1;
        }
        const int tt = p.tile0 + ((MC && t >= p.total_tiles) ? p.total_tiles - 1 : t);  // MC dummy: last tile
        const int b = MC ? 0 : tt / p.tiles_per_batch;
        const int row0 = (tt - b * p.tiles_per_batch) * (2 * BM) + rank * BM;
        mbar_wait(&a_empty[slot], aph ^ 1);
        // debug mode 3: event 5 records when this row tile's X load is issued
        if (dbg_mode(p) == 3 && pair == 0 && leader && lane == 0) trace_ev(p, (uint32_t)(j * p.ncol), 5);
        if (dbg_mode(p) == 7 && j >= a_slots) {  // bound analysis: X tiles loaded once per slot
          if (elect_one() && leader) mbar_arrive(&a_full[slot]);
          __syncwarp();
          continue;
        }
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&a_full[slot], 2 * a_bytes);
          const uint32_t bar = mapa_shared(smem_u32(&a_full[slot]), lead);
          for (int ka = 0; ka < p.katoms; ++ka)
            tma_load_3d_cg2(sA + slot * a_slot_bytes + ka * A_ATOM, &tmx, bar, ka * 64, row0, b,
                            FK_X_HINT);
        }
        __syncwarp();
      }
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ pair MMA (leader only)
    // The whole warp runs the loop so descriptor arithmetic stays warp-uniform
    // (uniform datapath); one elected lane issues each tcgen05 instruction.
    if (leader) {
      const uint32_t idesc = make_idesc_f16(FMT, 2 * BM, BN);
      const uint32_t idesc_main = NEG ? (idesc | kIdescNegateA) : idesc;
      const uint32_t idesc_ext = make_idesc_f16(1, 2 * BM, BN);
      const uint64_t aext_desc = make_sdesc_sw32(smem_u32(sAext));
      uint32_t stage = 0, sphase = 0, g = 0;
      int aslot = 0;
      uint32_t aphase = 0;
      for (int t = t_first; t < t_end; t += t_step) {
        const int slot = aslot;  // i % a_slots, without a division per tile
        const uint32_t aph = aphase;
        if (++aslot == a_slots) {
          aslot = 0;
          aphase ^= 1;
        }
        mbar_wait(&a_full[slot], aph);
        tc_fence_after();
        if (pair == 0 && lane == 0) trace_ev(p, g, 7);
        const uint32_t a_base = smem_u32(sA + slot * a_slot_bytes);
        for (int c = 0; c < p.ncol; ++c, ++g) {
          const uint32_t buf = g % NBUF;
          if (pair == 0 && lane == 0) trace_ev(p, g, 6);
          // SEED: every use of a buffer (the first two included) waits for its seed
          mbar_wait(&t_empty[buf], SEED ? ((g / NBUF) & 1) : (((g / NBUF) & 1) ^ 1));
          tc_fence_after();
          if (pair == 0 && lane == 0) trace_ev(p, g, 0);
          const uint32_t d_tmem = tmem_base + buf * BN;
          for (int ka = 0; ka < p.katoms; ++ka) {
            mbar_wait(&b_full[stage], sphase);
            tc_fence_after();
            const uint64_t adesc = make_sdesc_sw128(a_base + ka * A_ATOM);
            const uint64_t bdesc = make_sdesc_sw128(smem_u32(sB + stage * B_STAGE));
            if (elect_one()) {
              if constexpr (SPLIT) {
                // C step sc = 4 ka + k of the [c_hi | c_lo] row: c_hi steps meet
                // x_hi and x_lo, c_lo steps meet x_hi (x_lo . c_lo is dropped)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const int sc = 4 * ka + k;
                  if (sc < 2 * p.ns && dbg_mode(p) != 2) {
                    const int sa = sc < p.ns ? sc : sc - p.ns;
                    const uint64_t ad = make_sdesc_sw128(a_base + (sa >> 2) * A_ATOM) + 2 * (sa & 3);
                    tc_mma_f16_cg2(d_tmem, ad, bdesc + 2 * k, idesc_main, sc != 0);
                    if (sc < p.ns) {
                      const int sl = sc + p.ns;
                      const uint64_t al = make_sdesc_sw128(a_base + (sl >> 2) * A_ATOM) + 2 * (sl & 3);
                      tc_mma_f16_cg2(d_tmem, al, bdesc + 2 * k, idesc_main, 1u);
                    }
                  }
                }
              } else if (dbg_mode(p) != 2) {
#pragma unroll
                for (int k = 0; k < 4; ++k)  // +32 B along K = +2 in the descriptor's address field
                  tc_mma_f16_cg2(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc_main,
                                 SEED || (ka | k) != 0);
              }
              tc_commit_cg2_mc(&b_empty[stage], MC ? (uint16_t)0xF : pmask);  // MC: both pairs' producers
              // the row tile's last read of its X slot: release it now, ahead
              // of the bias step and the accumulator commit
              if (c == p.ncol - 1 && ka == p.katoms - 1) tc_commit_cg2_mc(&a_empty[slot], pmask);
            }
            __syncwarp();
            if (++stage == b_stages) {
              stage = 0;
              sphase ^= 1;
            }
          }
          if (AUG) {
            const uint32_t es = g % EXT_SLOTS;
            mbar_wait(&ext_full[es], (g / EXT_SLOTS) & 1);
            tc_fence_after();
            const uint64_t edesc = make_sdesc_sw32(smem_u32(sExt + es * EXT_SLOT));
            if (elect_one()) {
              tc_mma_f16_cg2(d_tmem, aext_desc, edesc, idesc_ext, dbg_mode(p) != 2 ? 1u : 0u);
              tc_commit_cg2_mc(&ext_empty[es], pmask);
            }
            __syncwarp();
          }
          if (elect_one()) tc_commit_cg2_mc(&t_full[buf], pmask);
          __syncwarp();
          if (pair == 0 && lane == 0) trace_ev(p, g, 1);
        }
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int wg = warp >> 2;        // column half of every tile (alt: tile parity)
    const int q = warp & 3;          // TMEM lane quarter
    const int row = q * 32 + lane;
    constexpr int nch = ALT ? 8 : 4;  // 32-column chunks this warp reads per tile
    // SEED: write ||c||^2/2 of pair-tile g2 (all rows alike) into TMEM buffer
    // g2 % NBUF, then hand the buffer to the MMA.
    auto seed_and_release = [&](uint32_t g2) __attribute__((always_inline)) {
      const uint32_t sbuf = g2 % NBUF;
      const int i2 = (int)(g2 / p.ncol);
      if (t_first + i2 * t_step < t_end && (!alt || (i2 & 1) == wg)) {
        const uint32_t cs = g2 % CN_SLOTS;
        mbar_wait(&cn_full[cs], (g2 / CN_SLOTS) & 1);
        const uint32_t src = smem_u32(sCN + cs * BN + (alt ? 0 : wg * (BN / 2)));
        const uint32_t saddr =
            tmem_base + (uint32_t(q * 32) << 16) + sbuf * BN + (alt ? 0 : wg * (BN / 2));
#pragma unroll 4
        for (int k = 0; k < 4 * nch; ++k) {  // 8 columns per store: few live registers
          const float4 f0 = lds128(src + 32 * k), f1 = lds128(src + 32 * k + 16);
          const uint32_t v[8] = {__float_as_uint(f0.x), __float_as_uint(f0.y), __float_as_uint(f0.z),
                                 __float_as_uint(f0.w), __float_as_uint(f1.x), __float_as_uint(f1.y),
                                 __float_as_uint(f1.z), __float_as_uint(f1.w)};
          tmem_st_x8(saddr + 8 * k, v);
        }
        tmem_wait_st();
        __syncwarp();
        if (lane == 0) mbar_arrive(&cn_empty[cs]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&t_empty[sbuf]);
        else
          mbar_arrive_cluster(mapa_shared(smem_u32(&t_empty[sbuf]), lead));
      }
    };
    if (SEED) {
      // the first use of each buffer; ALT: a warpgroup seeds only its own tiles
      for (uint32_t g0 = 0; g0 < NBUF; ++g0)
        if (!alt || (int)(g0 & 1) == wg) seed_and_release(g0);
    }
    uint32_t g = 0;
    int i = 0, aslot = 0;
    // (batch, tile-in-batch) of t, advanced without a division per tile
    int tb = (p.tile0 + t_first) / p.tiles_per_batch, tr_ = p.tile0 + t_first - tb * p.tiles_per_batch;
    const int step_b = t_step / p.tiles_per_batch, step_r = t_step - step_b * p.tiles_per_batch;
    for (int t = t_first; t < t_end; t += t_step, ++i) {
      const bool dummy = MC && t >= p.total_tiles;  // MC: keeps the C stream in step, writes nothing
      const int b = MC ? 0 : tb, trow = tr_;
      tb += step_b;
      tr_ += step_r;
      if (tr_ >= p.tiles_per_batch) {
        tr_ -= p.tiles_per_batch;
        ++tb;
      }
      const int slot = aslot;  // i % a_slots, without a division per tile
      if (++aslot == a_slots) aslot = 0;
      if (alt && (i & 1) != wg) {  // the other warpgroup owns this tile
        ++g;
        continue;
      }
      const int row0 = trow * (2 * BM) + rank * BM;
      // previous assignment of this row, loaded now so its HBM latency overlaps
      // the row tile's chunks instead of sitting at the end of the tile
      int prev_id = -2;
      if (p.idx_prev && (alt || wg == 0) && !dummy && row0 + row < p.N)
        prev_id = __ldg(p.idx_prev + (size_t)b * p.N + row0 + row);
      float xn_pre = 0.f;  // the precomputed ||x||^2 (owner warpgroup; the other adds 0)
      if (!SPLIT && p.xn_in && (alt || wg == 0) && !dummy && row0 + row < p.N)
        xn_pre = __ldg(p.xn_in + (size_t)b * p.N + row0 + row);
      float M = __int_as_float(0x7f800000);
      float m2 = M;  // split: lower bound on the row's second-best score
      float smg = 0.f;  // split: certificate margin of this row
      bool rovf = false;  // split: more near chunks than slots at some point
      int rec[SPLIT_NREC];  // near chunks: column base (-1 = free) and chunk minimum
      float rmn[SPLIT_NREC];
#pragma unroll
      for (int r = 0; r < SPLIT_NREC; ++r) {
        rec[r] = -1;
        rmn[r] = 0.f;
      }
      float cmx = 0.f;
      if (SPLIT) cmx = __uint_as_float(p.cmax[b]);
      int best = -1;
      float bestv[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) bestv[j] = M;
      float xn = 0.f;
      for (int c = 0; c < p.ncol; ++c, ++g) {
        const uint32_t buf = g % NBUF;
        const uint32_t cslot = g % CN_SLOTS;
        const bool tr = pair == 0 && leader && warp == 0 && lane == 0;
        mbar_wait(&t_full[buf], (g / NBUF) & 1);
        tc_fence_after();
        if (tr) trace_ev(p, g, 2);
        const uint32_t taddr =
            tmem_base + (uint32_t(q * 32) << 16) + buf * BN + (alt ? 0 : wg * (BN / 2));
        uint32_t va[32], vb[32];
        FK_TMEM_LD_32x32b_X32(taddr, va);
        if (c == 0) {  // ALT: the owning warpgroup; else each warpgroup half the chunk positions
          if (SPLIT) {  // |x| upper bound -> this row's certificate margin (k_certify's formula)
            xn = split_norm_ub(sA + slot * a_slot_bytes, row, p.katoms, p.ns, lane);
            smg = 0x1p-11f * fmaf(xn, cmx, cmx * cmx) + 0x1p-18f * xn * xn + 0x1p-100f;
            smg *= 1.0f + 0x1p-20f;
          } else if (p.xn_in) {
            xn = xn_pre;
          } else {
            xn = alt ? row_norm_smem<FMT>(sA + slot * a_slot_bytes, row, p.katoms, lane)
                     : row_norm_smem<FMT>(sA + slot * a_slot_bytes, row, p.katoms, lane, 4 * wg,
                                          4 * wg + 4);
          }
          __syncwarp();
          if (lane == 0 && (SPLIT || !p.xn_in)) mbar_arrive(&a_empty[slot]);
        }
        uint32_t cnp = 0;
        if (EPI) {
          mbar_wait(&cn_full[cslot], (g / CN_SLOTS) & 1);
          cnp = smem_u32(sCN + cslot * BN + (alt ? 0 : wg * (BN / 2)));
        }
        const int col0 = c * BN + (alt ? 0 : wg * (BN / 2));
        auto release_tmem = [&]() {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader)
              mbar_arrive(&t_empty[buf]);
            else
              mbar_arrive_cluster(mapa_shared(smem_u32(&t_empty[buf]), lead));
          }
        };
        // split: keep the chunk if its minimum is within the margin of the
        // running best (every centroid the exact argmin could be, or tie with)
        // (slots whose chunk minimum fell out of the margin of the current
        // best are freed first: the best only decreases)
        auto near = [&](float mc, int colbase) {
          if (SPLIT && mc <= M + smg) {
            bool put = false;
#pragma unroll
            for (int r = 0; r < SPLIT_NREC; ++r) {
              if (rec[r] >= 0 && rmn[r] > M + smg) rec[r] = -1;
              if (!put && rec[r] < 0) {
                rec[r] = colbase;
                rmn[r] = mc;
                put = true;
              }
            }
            rovf |= !put;
          }
        };
        auto chunk = [&](uint32_t (&v)[32], int ch) {
          if (NEG) {
            float mc = 0.f;
            epi_chunk_aug<SPLIT>(v, col0 + 32 * ch, M, best, bestv, m2, mc);
            near(mc, col0 + 32 * ch);
          } else
            epi_chunk(v, cnp + 128 * ch, col0 + 32 * ch, M, best, bestv);
        };
        if (dbg_mode(p) == 1) {
          FK_TMEM_WAIT_LD(va);
          release_tmem();  // (debug mode 1 does not support SEED: garbage accumulators are fine for timing)
          if (EPI && lane == 0) mbar_arrive(&cn_empty[cslot]);
          M = fminf(M, __uint_as_float(va[0]));
          continue;
        }
        if (AUG && p.epi2) {
          // chunk pairs: both loads in flight, one vote per pair
          FK_TMEM_LD_32x32b_X32(taddr + 32, vb);
#pragma unroll
          for (int ch = 0; ch < nch; ch += 2) {
            FK_TMEM_WAIT_LD(va);
            FK_TMEM_WAIT_LD(vb);
            if (ch + 2 >= nch) {
              release_tmem();  // every TMEM read of this buffer has landed
              if (tr) trace_ev(p, g, 3);
            }
            float mca = 0.f, mcb = 0.f;
            epi_chunk2_aug<SPLIT>(va, vb, col0 + 32 * ch, col0 + 32 * (ch + 1), M, best, bestv, m2, mca,
                                  mcb);
            near(mca, col0 + 32 * ch);
            near(mcb, col0 + 32 * (ch + 1));
            if (ch + 2 < nch) {
              FK_TMEM_LD_32x32b_X32(taddr + 32 * (ch + 2), va);
              FK_TMEM_LD_32x32b_X32(taddr + 32 * (ch + 3), vb);
            }
          }
          if (tr) trace_ev(p, g, 4);
          continue;
        }
#pragma unroll
        for (int ch = 0; ch < nch; ch += 2) {
          FK_TMEM_WAIT_LD(va);
          FK_TMEM_LD_32x32b_X32(taddr + 32 * (ch + 1), vb);
          chunk(va, ch);
          FK_TMEM_WAIT_LD(vb);
          if (ch + 2 < nch) {
            FK_TMEM_LD_32x32b_X32(taddr + 32 * (ch + 2), va);
          } else if (!SEED) {
            release_tmem();  // every TMEM read of this buffer has landed
            if (tr) trace_ev(p, g, 3);
          }
          chunk(vb, ch + 1);
        }
        if (SEED) {
          seed_and_release(g + NBUF);  // reads done: seed the tile that reuses this buffer
          if (tr) trace_ev(p, g, 3);
        }
        if (tr) trace_ev(p, g, 4);
        if (EPI) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&cn_empty[cslot]);
        }
      }
      int idx = -1;
      if (best >= 0) {
        int found = 31;
#pragma unroll
        for (int j = 31; j >= 0; --j) found = (bestv[j] == M) ? j : found;
        idx = best + found;
        if constexpr (SPLIT) {  // the rest of the winning chunk
#pragma unroll
          for (int j = 0; j < 32; ++j) m2 = j != found ? fminf(m2, bestv[j]) : m2;
        }
      }
      int nrec = 0;  // split: the near chunks still within the margin of this half's best
      if constexpr (SPLIT) {
#pragma unroll
        for (int r = 0; r < SPLIT_NREC; ++r) {
          if (rec[r] >= 0 && rmn[r] > M + smg) rec[r] = -1;
          nrec += rec[r] >= 0 ? 1 : 0;
        }
        if (rovf) nrec = SPLIT_NREC + 1;
      }
      if (!alt) {
        if (wg == 1) {
          xch_m[row] = M;
          xch_i[row] = idx;
          xch_xn[row] = xn;
          if (SPLIT) {
            xch_m2[row] = m2;
            xch_rec[row * 8] = nrec;
            int w8 = 0;
#pragma unroll
            for (int r = 0; r < SPLIT_NREC; ++r)
              if (rec[r] >= 0) xch_rec[row * 8 + 1 + w8++] = rec[r];
          }
        }
        named_bar_sync(1, 256);
        if (wg == 0) {
          if (!SPLIT) xn += xch_xn[row];
          const float M1 = xch_m[row];
          const int i1 = xch_i[row];
          if (SPLIT) m2 = fminf(fminf(m2, xch_m2[row]), fmaxf(M, M1));
          if (M1 < M || (M1 == M && i1 >= 0 && (idx < 0 || i1 < idx))) {
            M = M1;
            idx = i1;
          }
        }
      }
      if (alt || wg == 0) {
        const int grow = row0 + row;
        bool ch = false;
        if (!dummy && grow < p.N) {
          const size_t o = (size_t)b * p.N + grow;
          p.idx_out[o] = idx;
          if (SPLIT) {  // raw scores: the certify pass decides and computes the distance
            p.mind_out[o] = M;
            p.second_out[o] = m2;
          } else {
            p.mind_out[o] = fmaxf(0.f, NEG ? fmaf(2.f, M, xn) : xn + M);
            if (p.idx_prev) ch = prev_id != idx;
            if (p.hist_tab) {  // fire-and-forget reductions (RED), integer: order-free
              const int64_t r = (int64_t)b * p.hist_bpb + grow / p.hist_per;
              if (idx >= 0 && idx < p.K)
                atomicAdd(p.hist_tab + r * p.K + idx, 1);
              else
                atomicAdd(p.hist_inval + r, 1);
            }
          }
        }
        if (p.changed && __any_sync(0xffffffffu, ch) && lane == 0) atomicOr(p.changed, 1);
        if constexpr (SPLIT) {
          // the epilogue's certificate (margin >= k_certify's: |x| bounded from
          // above), else the near chunks of both column halves, else a full
          // fallback; records appended warp-aggregated
          const int n1 = alt ? 0 : xch_rec[row * 8];
          const float scale = fmaf(xn, cmx, cmx * cmx);
          const bool cert = idx >= 0 && (m2 - M > smg) && scale > 0x1p-60f && smg < 3e38f;
          const bool live = grow < p.N;
          const bool lst = live && !cert && nrec <= SPLIT_NREC && n1 <= SPLIT_NREC && smg < 3e38f;
          const unsigned m = __ballot_sync(0xffffffffu, lst);
          int pos = -1;
          if (m) {
            int base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(p.cand_cnt, __popc(m));
            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
            if (lst) pos = base + __popc(m & ((1u << lane) - 1));
          }
          const bool listed = lst && pos < p.cand_cap;
          if (listed) {
            int32_t* r = p.cand_rec + (int64_t)pos * FK_SPLIT_REC;
            r[0] = (int32_t)((int64_t)b * p.N + grow);
            const int n0 = nrec;  // <= SPLIT_NREC here
            r[1] = n0 + n1;
            int w8 = 0;
#pragma unroll
            for (int q2 = 0; q2 < SPLIT_NREC; ++q2)
              if (rec[q2] >= 0) r[2 + w8++] = rec[q2];
            for (int q2 = 0; q2 < n1; ++q2) r[2 + n0 + q2] = xch_rec[row * 8 + 1 + q2];
          }
          if (live) p.stat_out[(size_t)b * p.N + grow] = cert ? 0 : (listed ? 1 : 2);
        }
      }
      if (!alt) named_bar_sync(2, 256);
    }
    tc_fence_before();
  }
  cluster_sync();
  if (warp == W_TMEM) {
    tc_fence_after();
    tmem_dealloc_cg2<512>(tmem_base);
  }
}

template <int FMT, int BIAS, bool ALT, bool SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc2::THREADS, 1)
    fk_assign_tc2_kernel(const __grid_constant__ CUtensorMap tmx,
                         const __grid_constant__ CUtensorMap tmc,
                         const __grid_constant__ CUtensorMap tmext, const TcArgs p) {
  assign_tc2_body<FMT, BIAS, ALT, SPLIT, false>(tmx, tmc, tmext, p);
  // launched beside the multicast quads (programmatic dependent launch): do
  // not complete before them, so stream order after this kernel covers both
  // (a no-op for an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Two CTA pairs per cluster sharing the C stream by multicast (see MC above).
template <int FMT>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(tc2::THREADS, 1)
    fk_assign_tc2q_kernel(const __grid_constant__ CUtensorMap tmx,
                          const __grid_constant__ CUtensorMap tmc,
                          const __grid_constant__ CUtensorMap tmext, const TcArgs p) {
  // every quad is resident from the start: release the pair kernel that
  // takes the SMs the 4-CTA clusters cannot use
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  assign_tc2_body<FMT, 1, false, false, true>(tmx, tmc, tmext, p);
}

template <int FMT, int BIAS, bool ALT, bool SPLIT = false>
static cudaError_t launch_pair_t(const CUtensorMap& tmx, const CUtensorMap& tmc,
                                 const CUtensorMap& tmext, TcArgs a, int pairs,
                                 cudaStream_t stream) {
  static int attr_dev_mask = 0;  // one-time per device (keeps graph capture free of it)
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_dev_mask & (1 << (dev & 31)))) {
    cudaFuncSetAttribute(fk_assign_tc2_kernel<FMT, BIAS, ALT, SPLIT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, tc2::SMEM_BYTES);
    attr_dev_mask |= 1 << (dev & 31);
  }
  fk_assign_tc2_kernel<FMT, BIAS, ALT, SPLIT><<<2 * pairs, tc2::THREADS, tc2::SMEM_BYTES, stream>>>(
      tmx, tmc, tmext, a);
  return cudaGetLastError();
}

// Multicast quads (fk_assign_tc2q_kernel): launched as many 4-CTA clusters as
// fit at once (a GPC whose SM count is not a multiple of 4 leaves SMs idle),
// at most one per tile pair.
template <int FMT>
static cudaError_t launch_quad(const CUtensorMap& tmx, const CUtensorMap& tmc,
                               const CUtensorMap& tmc_pair, const CUtensorMap& tmext, TcArgs a,
                               int num_sms, cudaStream_t stream) {
  static int quads_dev[32] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = fk_assign_tc2q_kernel<FMT>;
  auto pk = fk_assign_tc2_kernel<FMT, 1, false, false>;
  int& fit = quads_dev[dev & 31];
  if (fit == 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tc2::SMEM_BYTES);
    cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, tc2::SMEM_BYTES);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(num_sms & ~3));
    cfg.blockDim = dim3(tc2::THREADS);
    cfg.dynamicSmemBytes = tc2::SMEM_BYTES;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = num_sms / 4;
    }
    fit = n;
    if (getenv("FK_ASSIGN_MC_VERBOSE"))
      fprintf(stderr, "fk_assign_tc2q: %d co-resident 4-CTA clusters (%d SMs)\n", n, num_sms);
  }
  a.tiles_per_batch = (a.N + 2 * tc2::BM - 1) / (2 * tc2::BM);
  a.total_tiles = a.B * a.tiles_per_batch;
  a.ncol = (a.K + tc2::BN - 1) / tc2::BN;
  const int total = a.total_tiles;
  int quads = fit;
  if ((total + 1) / 2 < quads) quads = (total + 1) / 2;
  if (quads <= 0) return cudaSuccess;
  // the SMs no 4-CTA cluster can use run the pair kernel on the tiles after
  // the quads' share, sized by the quads' measured per-SM advantage
  int extra = (num_sms - 4 * fit) / 2;
  {
    static int extra_env = -2;
    if (extra_env == -2) {
      const char* e = getenv("FK_ASSIGN_MC_EXTRA");
      extra_env = e ? atoi(e) : -1;
    }
    if (extra_env >= 0 && extra_env < extra) extra = extra_env;
  }
  int tq = total;
  if (extra > 0 && quads == fit && total >= 8 * (quads + extra)) {
    static double gain = -1.0;
    if (gain < 0) {
      const char* e = getenv("FK_ASSIGN_MC_GAIN");
      gain = e ? atof(e) : 1.12;
    }
    const double wq = 4.0 * quads * gain, wp = 2.0 * extra;
    tq = ((int)(total * wq / (wq + wp)) + 1) & ~1;
    if (tq > total) tq = total;
  } else {
    extra = 0;
  }
  TcArgs aq = a;
  aq.total_tiles = tq;
  kern<<<4 * quads, tc2::THREADS, tc2::SMEM_BYTES, stream>>>(tmx, tmc, tmext, aq);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess || tq >= total) return err;
  TcArgs ap = a;
  ap.tile0 = tq;
  ap.total_tiles = total - tq;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * extra));
  cfg.blockDim = dim3(tc2::THREADS);
  cfg.dynamicSmemBytes = tc2::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, pk, tmx, tmc_pair, tmext, ap);
}

// FK_ASSIGN_MC=1: multicast quads where they apply (A/B switch)
static bool assign_mc_enabled() {
  static int mc_env = -1;
  if (mc_env < 0) {
    const char* e = getenv("FK_ASSIGN_MC");
    mc_env = (e && e[0] == '1') ? 1 : 0;
  }
  return mc_env == 1;
}

// Rows of a single column tile (K <= 256) alternate tiles between the two
// epilogue warpgroups; FK_ASSIGN_ALT=0 splits their columns instead (A/B)
static bool pair_alt(int K) {
  static int alt_env = -1;
  if (alt_env < 0) {
    const char* e = getenv("FK_ASSIGN_ALT");
    alt_env = (e && e[0] == '0') ? 0 : 1;
  }
  return (K + tc2::BN - 1) / tc2::BN == 1 && alt_env;
}

template <int FMT, int BIAS>
static cudaError_t launch_pair(const CUtensorMap& tmx, const CUtensorMap& tmc,
                               const CUtensorMap& tmext, TcArgs a, int num_sms,
                               cudaStream_t stream) {
  a.tiles_per_batch = (a.N + 2 * tc2::BM - 1) / (2 * tc2::BM);
  a.total_tiles = a.B * a.tiles_per_batch;
  a.ncol = (a.K + tc2::BN - 1) / tc2::BN;
  int pairs = num_sms / 2;
  if (a.total_tiles < pairs) pairs = a.total_tiles;
  if (pairs <= 0) return cudaSuccess;
  return pair_alt(a.K) ? launch_pair_t<FMT, BIAS, true>(tmx, tmc, tmext, a, pairs, stream)
                       : launch_pair_t<FMT, BIAS, false>(tmx, tmc, tmext, a, pairs, stream);
}

// ---------------------------------------------------- row norms, epilogue order
// ||x||^2 of every row exactly as the pair kernel's epilogue sums it from the
// 128-byte-swizzled shared tile (row_norm_smem): lane = row % 32 reads
// physical 16-byte chunk (j + lane) & 7, i.e. logical chunk
// ((j + lane) & 7) ^ (row & 7), atoms in order, element pairs (lo, hi) by
// fmaf; columns beyond d are the tile's zero fill.  ALT (one column tile):
// one sum over j = 0..7; otherwise the two warpgroups' halves (j < 4, j >= 4)
// added (wg0 + wg1) as the epilogue's merge does.
template <int FMT>
__global__ void __launch_bounds__(256)
    k_row_norms_tc(const uint16_t* __restrict__ X, int64_t rows, int64_t N, int d, int alt,
                   float* __restrict__ out) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int grow = (int)(r % N);
  const int lane = grow & 31, sw = grow & 7;
  const uint4* xr = reinterpret_cast<const uint4*>(X + r * d);  // rows are 16-byte multiples
  const int katoms = (d + 63) / 64;
  auto part = [&](int j0, int j1) {
    float acc = 0.f;
    for (int ka = 0; ka < katoms; ++ka)
      for (int j = j0; j < j1; ++j) {
        const int lc = ka * 8 + (((j + lane) & 7) ^ sw);  // 16-byte chunk of the row
        if (8 * lc >= d) continue;  // the tile's zero fill: fmaf(0, 0, acc) == acc
        const uint4 w = __ldg(xr + lc);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float lo, hi;
          if (FMT == 1) {
            lo = __uint_as_float(ws[e] << 16);
            hi = __uint_as_float(ws[e] & 0xffff0000u);
          } else {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&ws[e]));
            lo = f.x;
            hi = f.y;
          }
          acc = fmaf(lo, lo, acc);
          acc = fmaf(hi, hi, acc);
        }
      }
    return acc;
  };
  out[r] = alt ? part(0, 8) : part(0, 4) + part(4, 8);
}

cudaError_t launch_row_norms_tc(int fmt, const void* X, int64_t B, int64_t N, int64_t K, int64_t d,
                                float* out, cudaStream_t stream) {
  const int64_t rows = B * N;
  if (rows < 1) return cudaSuccess;
  const unsigned grid = (unsigned)((rows + 255) / 256);
  const int alt = pair_alt((int)K) ? 1 : 0;
  if (fmt == 1)
    k_row_norms_tc<1><<<grid, 256, 0, stream>>>((const uint16_t*)X, rows, N, (int)d, alt, out);
  else
    k_row_norms_tc<0><<<grid, 256, 0, stream>>>((const uint16_t*)X, rows, N, (int)d, alt, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D map over (inner, rows, B): box {box_inner, box_rows, 1}; 128-B swizzle
// for the 64-wide K atoms of X / C, 32-B swizzle for the 16-wide bias operand.
static bool make_map(CUtensorMap* m, const void* base, int fmt, int64_t inner, int64_t rows,
                     int64_t B, int box_rows, int box_inner = 64,
                     CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)B};
  cuuint64_t strides[2] = {(cuuint64_t)(inner * 2), (cuuint64_t)(rows * inner * 2)};
  cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, fmt == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, FK_TMAP_PROMO,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

constexpr int kDefaultBiasMode = 1;

bool assign_tc_supported(int64_t d) { return d >= 8 && d <= 256 && (d % 8) == 0; }

// Where the ||c||^2/2 bias enters (FK_ASSIGN_BIAS=0 epilogue, 1 bias-in-GEMM,
// 2 TMEM seed; A/B comparisons).  The legacy FK_ASSIGN_AUG=0 means 0.
int assign_tc_bias_mode(int fmt) {
  (void)fmt;
  const char* e = getenv("FK_ASSIGN_BIAS");
  if (e && e[0] >= '0' && e[0] <= '2') return e[0] - '0';
  const char* a = getenv("FK_ASSIGN_AUG");
  if (a && atoi(a) == 0) return 0;
  return kDefaultBiasMode;
}
bool assign_tc_uses_ext(int fmt) { return assign_tc_bias_mode(fmt) == 1; }

cudaError_t launch_assign_tc(int fmt, const void* X, const void* C, const float* cn_pad,
                             const void* cn_ext, int64_t B, int64_t N, int64_t K, int64_t d,
                             int32_t* idx_out, float* mind_out, const int32_t* idx_prev,
                             int32_t* changed, int num_sms, cudaStream_t stream, int32_t* hist_tab,
                             int32_t* hist_inval, int64_t hist_bpb, int64_t hist_per,
                             const float* xn_in) {
  TcArgs a;
  a.tile0 = 0;
  a.xn_in = xn_in;
  a.hist_tab = hist_tab;
  a.hist_inval = hist_inval;
  a.hist_bpb = (int)hist_bpb;
  a.hist_per = (int)(hist_per < 1 ? 1 : hist_per);
  a.B = (int)B;
  a.N = (int)N;
  a.K = (int)K;
  a.d = (int)d;
  a.katoms = (int)((d + 63) / 64);
  a.tiles_per_batch = (int)((N + tc::BM - 1) / tc::BM);
  a.total_tiles = (int)(B * a.tiles_per_batch);
  a.ncol = (int)((K + tc::BN - 1) / tc::BN);
  a.kpad = a.ncol * tc::BN;
  a.cn = cn_pad;
  a.idx_out = idx_out;
  a.mind_out = mind_out;
  a.idx_prev = idx_prev;
  a.changed = changed;
  {
    const char* dm = getenv("FK_ASSIGN_DEBUG_MODE");
    a.debug_mode = dm ? atoi(dm) : 0;
    // chunk pairs help when row tiles are short (K <= 1024: +1.5-3% at configs
    // 2 and 4) and cost ~3% at K = 4096 (same-box A/B, profiles/r01_ab_epi2.txt)
    const char* e2 = getenv("FK_ASSIGN_EPI2");
    a.epi2 = e2 ? (e2[0] == '1') : (a.ncol <= 4);
  }
  a.trace = nullptr;
  a.ns = 0;
  a.second_out = nullptr;
  static unsigned long long* trace_buf = nullptr;
  const char* trace_path = getenv("FK_ASSIGN_TRACE");
  if (trace_path) {
    if (!trace_buf) cudaMalloc(&trace_buf, TR_N * TR_EV * 8);
    cudaMemsetAsync(trace_buf, 0, TR_N * TR_EV * 8, stream);
    a.trace = trace_buf;
  }
  const char* cta = getenv("FK_ASSIGN_CTA");
  if (!(cta && atoi(cta) == 1) || d > 128) {  // the single-CTA kernel (A/B only) stops at d = 128
    CUtensorMap tmx2, tmc2, tmext;
    if (!make_map(&tmx2, X, fmt, d, N, B, tc2::BM)) return cudaErrorInvalidValue;
    if (!make_map(&tmc2, C, fmt, d, K, B, tc2::BNH)) return cudaErrorInvalidValue;
    const int bias = cn_ext != nullptr ? 1 : (assign_tc_bias_mode(fmt) == 2 ? 2 : 0);
    const bool aug = bias == 1;
    if (aug) {
      if (!make_map(&tmext, cn_ext, 1, 16, a.kpad, B, tc2::BNH, 16, CU_TENSOR_MAP_SWIZZLE_32B))
        return cudaErrorInvalidValue;
    } else {
      tmext = tmc2;  // unused
    }
    cudaError_t e;
    const bool mc = bias == 1 && B == 1 && a.ncol >= 2 && assign_mc_enabled();
    CUtensorMap tmcq;
    if (mc && !make_map(&tmcq, C, fmt, d, K, B, tc2::BNH / 2)) return cudaErrorInvalidValue;
    if (mc)
      e = fmt == 1 ? launch_quad<1>(tmx2, tmcq, tmc2, tmext, a, num_sms, stream)
                   : launch_quad<0>(tmx2, tmcq, tmc2, tmext, a, num_sms, stream);
    else if (fmt == 1)
      e = bias == 1   ? launch_pair<1, 1>(tmx2, tmc2, tmext, a, num_sms, stream)
          : bias == 2 ? launch_pair<1, 2>(tmx2, tmc2, tmext, a, num_sms, stream)
                      : launch_pair<1, 0>(tmx2, tmc2, tmext, a, num_sms, stream);
    else
      e = bias == 1   ? launch_pair<0, 1>(tmx2, tmc2, tmext, a, num_sms, stream)
          : bias == 2 ? launch_pair<0, 2>(tmx2, tmc2, tmext, a, num_sms, stream)
                      : launch_pair<0, 0>(tmx2, tmc2, tmext, a, num_sms, stream);
    if (trace_path && e == cudaSuccess) {  // debug only: synchronous dump
      unsigned long long h[TR_N * TR_EV];
      cudaMemcpyAsync(h, trace_buf, sizeof(h), cudaMemcpyDeviceToHost, stream);
      cudaStreamSynchronize(stream);
      FILE* f = fopen(trace_path, "w");
      if (f) {
        for (int i = 0; i < TR_N; ++i) {
          for (int j = 0; j < TR_EV; ++j) fprintf(f, "%llu ", h[i * TR_EV + j]);
          fprintf(f, "\n");
        }
        fclose(f);
      }
    }
    return e;
  }
  if (hist_tab || xn_in) return cudaErrorInvalidValue;  // the single-CTA A/B kernel: neither
  CUtensorMap tmx, tmc;
  if (!make_map(&tmx, X, fmt, d, N, B, tc::BM)) return cudaErrorInvalidValue;
  if (!make_map(&tmc, C, fmt, d, K, B, tc::BN)) return cudaErrorInvalidValue;
  const int grid = a.total_tiles < num_sms ? a.total_tiles : num_sms;
  if (grid <= 0) return cudaSuccess;
  if (fmt == 1) {
    cudaFuncSetAttribute(fk_assign_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         tc::SMEM_BYTES);
    fk_assign_tc_kernel<1><<<grid, tc::THREADS, tc::SMEM_BYTES, stream>>>(tmx, tmc, a);
  } else {
    cudaFuncSetAttribute(fk_assign_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         tc::SMEM_BYTES);
    fk_assign_tc_kernel<0><<<grid, tc::THREADS, tc::SMEM_BYTES, stream>>>(tmx, tmc, a);
  }
  return cudaGetLastError();
}

// Split operands (fk_assign_split.cu): X2 (B, N, 32 ns) and C2 (B, K, 32 ns)
// bf16 rows [hi (16 ns) | lo (16 ns)], bias operand ext (B, kpad, 16).
// Writes the estimated argmin ids, its score (||c||^2/2 - x.c) and a lower
// bound on the row's second-best score.
cudaError_t launch_assign_tc_split(const void* X2, const void* C2, const void* ext, int64_t B,
                                   int64_t N, int64_t K, int ns, int32_t* idx_out, float* est_out,
                                   float* second_out, const unsigned int* cmax, int8_t* stat_out,
                                   int32_t* cand_rec, int32_t* cand_cnt, int cand_cap, int num_sms,
                                   cudaStream_t stream) {
  if (ns < 1 || 2 * ns > 4 * tc2::KATOMS_MAX) return cudaErrorInvalidValue;
  const int64_t W = 32 * (int64_t)ns;
  TcArgs a;
  a.tile0 = 0;
  a.xn_in = nullptr;
  a.hist_tab = nullptr;
  a.hist_inval = nullptr;
  a.hist_bpb = 1;
  a.hist_per = 1;
  a.B = (int)B;
  a.N = (int)N;
  a.K = (int)K;
  a.d = (int)W;
  a.katoms = (int)((W + 63) / 64);
  a.ncol = (int)((K + tc::BN - 1) / tc::BN);
  a.kpad = a.ncol * tc::BN;
  a.cn = nullptr;
  a.idx_out = idx_out;
  a.mind_out = est_out;
  a.idx_prev = nullptr;
  a.changed = nullptr;
  {
    const char* dm = getenv("FK_ASSIGN_DEBUG_MODE");
    a.debug_mode = dm ? atoi(dm) : 0;
    const char* e2 = getenv("FK_ASSIGN_EPI2");
    a.epi2 = e2 ? (e2[0] == '1') : (a.ncol <= 4);
  }
  a.trace = nullptr;
  a.ns = ns;
  a.second_out = second_out;
  a.cmax = cmax;
  a.stat_out = stat_out;
  a.cand_rec = cand_rec;
  a.cand_cnt = cand_cnt;
  a.cand_cap = cand_cap;
  CUtensorMap tmx2, tmc2, tmext;
  if (!make_map(&tmx2, X2, 1, W, N, B, tc2::BM)) return cudaErrorInvalidValue;
  if (!make_map(&tmc2, C2, 1, W, K, B, tc2::BNH)) return cudaErrorInvalidValue;
  if (!make_map(&tmext, ext, 1, 16, a.kpad, B, tc2::BNH, 16, CU_TENSOR_MAP_SWIZZLE_32B))
    return cudaErrorInvalidValue;
  a.tiles_per_batch = (a.N + 2 * tc2::BM - 1) / (2 * tc2::BM);
  a.total_tiles = a.B * a.tiles_per_batch;
  int pairs = num_sms / 2;
  if (a.total_tiles < pairs) pairs = a.total_tiles;
  if (pairs <= 0) return cudaSuccess;
  return a.ncol == 1 ? launch_pair_t<1, 1, true, true>(tmx2, tmc2, tmext, a, pairs, stream)
                     : launch_pair_t<1, 1, false, true>(tmx2, tmc2, tmext, a, pairs, stream);
}

int assign_tc_kpad(int64_t K) { return (int)(((K + tc::BN - 1) / tc::BN) * tc::BN); }

FK_MODULE_ANCHOR(assign_tc)

}  // namespace fk
