// fk_common.cuh -- sm_100a PTX helpers shared by the flash-kmeans kernels.
// Hand-written inline PTX: mbarrier, TMA (cp.async.bulk.tensor), tcgen05
// (alloc / mma / commit / ld / fences).  No CUTLASS/CuTe code is used; the
// descriptor bit layouts follow the PTX ISA tables for sm_100a.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define FK_DEV __device__ __forceinline__

namespace fk {

// ------------------------------------------------------------------ smem
FK_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// -------------------------------------------------------------- mbarrier
FK_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
FK_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
FK_DEV void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
FK_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
FK_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
FK_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
FK_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ------------------------------------------------------------------- TMA
FK_DEV void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(desc) : "memory");
}
// 3-D tiled load global -> shared, completion signalled on `bar` (tx bytes).
FK_DEV void tma_load_3d(void* smem_dst, const void* desc, uint64_t* bar, int c0, int c1, int c2,
                        uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::"
      "cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(cache_hint)
      : "memory");
}
// 1-D bulk copy global -> shared (size and addresses multiples of 16 B).
FK_DEV void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 cache-policy constants (createpolicy.fractional.* encodings as used by CUTLASS).
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;
constexpr uint64_t kEvictNormal = 0x1000000000000000ull;

// --------------------------------------------------------------- tcgen05
template <int kCols>
FK_DEV void tmem_alloc(uint32_t* dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int kCols>
FK_DEV void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
FK_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
FK_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16/fp16 in, fp32 accumulate).
FK_DEV void tc_mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on `bar` once every previously issued tcgen05 op of this thread completes.
FK_DEV void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// Instruction descriptor, kind::f16: D=f32, A/B = bf16 (fmt 1) or f16 (fmt 0),
// both K-major, dense.  Bits: c_format[4,6)=1, a_format[7,10), b_format[10,13),
// a_major[15]=0, b_major[16]=0, n>>3 at [17,23), m>>4 at [24,29).
__host__ __device__ constexpr uint32_t make_idesc_f16(int fmt, int M, int N) {
  return (1u << 4) | (uint32_t(fmt) << 7) | (uint32_t(fmt) << 10) | (uint32_t(N >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}

// Shared-memory matrix descriptor: K-major operand stored by TMA with
// SWIZZLE_128B (rows of 128 B, 8-row / 1024 B swizzle atoms).
//   [0,14) start>>4  [16,30) LBO>>4 (unused for this layout)  [32,46) SBO>>4 = 1024>>4
//   [46,48) version=1  [49,52) base offset=0  [61,64) layout=2 (SWIZZLE_128B)
FK_DEV uint64_t make_sdesc_sw128(uint32_t smem_addr) {
  return uint64_t((smem_addr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// Same for a K-major operand whose rows are 32 B (16 bf16) wide, stored with
// SWIZZLE_32B (8-row / 256 B atoms): layout type 6, SBO = 256 B.
FK_DEV uint64_t make_sdesc_sw32(uint32_t smem_addr) {
  return uint64_t((smem_addr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(256 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(6) << 61);
}
constexpr uint32_t kIdescNegateA = 1u << 13;

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
#define FK_TMEM_LD_32x32b_X32(taddr, r)                                                          \
  asm volatile(                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"   \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"         \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),     \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),           \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),           \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])            \
      : "r"(taddr)                                                                               \
      : "memory")

// Wait for outstanding tcgen05.ld of this thread.  The registers are passed
// as read-write operands so the compiler cannot hoist their uses above it.
#define FK_TMEM_WAIT_LD(r)                                                                      \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                 \
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),       \
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),     \
                 "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), \
                 "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), \
                 "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), \
                 "+r"(r[30]), "+r"(r[31])                                                     \
               :                                                                                \
               : "memory")

// Register -> TMEM store: each lane writes 32 consecutive columns of its lane.
#define FK_TMEM_ST_32x32b_X32(taddr, r)                                                          \
  asm volatile(                                                                                  \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"            \
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),  \
      "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), \
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),        \
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),         \
      "r"(r[29]), "r"(r[30]), "r"(r[31])                                                          \
      : "memory")
FK_DEV void tmem_st_x8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
FK_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

FK_DEV float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

// ---------------------------------------------------------------- clusters
FK_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
FK_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
FK_DEV uint32_t mapa_shared(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
FK_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// 2-SM TMA: the bytes land in this CTA's smem; completion is counted on the
// mbarrier at `bar_cluster_addr` (the leader CTA's barrier).
FK_DEV void tma_load_3d_cg2(void* smem_dst, const void* desc, uint32_t bar_cluster_addr, int c0,
                            int c1, int c2, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::"
      "cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(desc), "r"(bar_cluster_addr), "r"(c0), "r"(c1), "r"(c2), "l"(cache_hint)
      : "memory");
}
// 2-SM TMA multicast: the box lands at the same offset in every CTA of `mask`;
// each destination's bytes are counted on the barrier at this offset in the
// leader of the destination's own pair (`bar_cluster_addr` names the leader of
// the issuing CTA's pair).
FK_DEV void tma_load_3d_cg2_mc(void* smem_dst, const void* desc, uint32_t bar_cluster_addr,
                               uint16_t mask, int c0, int c1, int c2, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes."
      "multicast::cluster.L2::cache_hint [%0], [%1, {%4, %5, %6}], [%2], %3, %7;" ::"r"(
          smem_u32(smem_dst)),
      "l"(desc), "r"(bar_cluster_addr), "h"(mask), "r"(c0), "r"(c1), "r"(c2), "l"(cache_hint)
      : "memory");
}
template <int kCols>
FK_DEV void tmem_alloc_cg2(uint32_t* dst_smem) {  // one warp in EACH CTA of the pair
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <int kCols>
FK_DEV void tmem_dealloc_cg2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
// Pair MMA (issued by the leader CTA only): D[256 x N] over both CTAs' TMEM.
FK_DEV void tc_mma_f16_cg2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Commit the leader's pair MMAs to the same-offset mbarrier in every CTA of `mask`.
FK_DEV void tc_commit_cg2_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// ------------------------------------------------------------- math bits
FK_DEV float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// (a.x,a.y) * s + (c.x,c.y) with one packed FFMA2.
FK_DEV float2 ffma2(float2 a, float2 s, float2 c) {
  uint64_t ra = *reinterpret_cast<uint64_t*>(&a), rs = *reinterpret_cast<uint64_t*>(&s),
           rc = *reinterpret_cast<uint64_t*>(&c), rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rs), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}

FK_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

FK_DEV uint32_t lane_id() {
  uint32_t l;
  asm("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

FK_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}


// ---------------------------------------------------------------------------
// numpy's float64 reduction order for np.sum(m, dtype=float64) of a float32
// row m (pipeline._objective_row, the objective of every non-f64 run): the
// ufunc machinery casts the row through its 8192-element buffer
// (np.getbufsize()) and adds each buffer's pairwise_sum_DOUBLE
// (numpy/_core/src/umath/loops_utils.h.src: leaves of <= 128 values summed by
// 8 interleaved accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
// above that a split at n/2 rounded down to a multiple of 8) into the running
// sum in buffer order.  np_pairwise_block reproduces one buffer's pairwise sum
// with a block of threads; the buffer sums are then folded in order from 0.0.
// (Pinned by tests/test_gpu_kernels.py against numpy on inexact data.)
constexpr int kNpBuf = 8192;
constexpr int kNpLeaf = 128;
constexpr int kNpDepth = 7;       // max recursion depth for n <= 8192
constexpr int kNpMaxLeaves = 72;  // max leaves for n <= 8192 is 65

__host__ __device__ inline int np_split(int n) {
  const int h = n >> 1;
  return h - (h & 7);
}

struct NpScratch {
  double V[(2 << kNpDepth) - 1];  // node values, heap order
  uint8_t kind[(2 << kNpDepth) - 1];  // 0 absent, 1 leaf, 2 internal
  int16_t leaf_lo[kNpMaxLeaves], leaf_n[kNpMaxLeaves], leaf_v[kNpMaxLeaves];
  int nleaf;
};

// Pairwise sum of src[0, n0) (n0 <= 8192, each value cast to double) by the
// whole block (every thread calls it; >= 64 threads); the result is returned
// to every thread.
template <typename T>
FK_DEV double np_leaf8(const T* __restrict__ src, int lo, int n, int sub) {
  // numpy's leaf (8 <= n <= 128 or shorter): lane `sub` of an 8-lane group is
  // accumulator r[sub]; its <= 16 loads issued before the serial adds
  const int body = n >= 8 ? n - (n % 8) : 0;
  double v[kNpLeaf / 8];
#pragma unroll
  for (int i = 0; i < kNpLeaf / 8; ++i) v[i] = 8 * i < body ? (double)src[lo + 8 * i + sub] : 0.0;
  double r = v[0];
#pragma unroll
  for (int i = 1; i < kNpLeaf / 8; ++i)
    if (8 * i < body) r = __dadd_rn(r, v[i]);
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
  double res = body > 0 ? r : 0.0;  // lane sub == 0 adds the tail
  if (sub == 0)
    for (int i = body; i < n; ++i) res = __dadd_rn(res, (double)src[lo + i]);
  return res;
}

template <typename T>
__device__ double np_pairwise_block(const T* __restrict__ src, int n0, NpScratch& s) {
  if (n0 == kNpBuf) {
    // a full buffer: 64 leaves of 128 under a perfect binary tree
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane & 7;
    const int nw = blockDim.x >> 5;
    for (int L0 = warp * 4; L0 < kNpBuf / kNpLeaf; L0 += nw * 4) {
      const int L = L0 + (lane >> 3);
      const double v = np_leaf8(src, L * kNpLeaf, kNpLeaf, sub);
      if (sub == 0) s.V[L] = v;
    }
    __syncthreads();
    if (warp == 0) {
      double x = __dadd_rn(s.V[2 * lane], s.V[2 * lane + 1]);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {  // left + right at every level
        const double y = __shfl_down_sync(0xffffffffu, x, o);
        if ((lane & (2 * o - 1)) == 0) x = __dadd_rn(x, y);
      }
      if (lane == 0) s.V[64] = x;
    }
    __syncthreads();
    return s.V[64];
  }
  if (threadIdx.x == 0) s.nleaf = 0;
  __syncthreads();
  // A: classify the nodes of the recursion tree (heap index), list the leaves
  for (int r = 0; r <= kNpDepth; ++r) {
    const int cnt = 1 << r;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
      int lo = 0, n = n0;
      bool exists = true;
      for (int t = r - 1; t >= 0; --t) {
        if (n <= kNpLeaf) {
          exists = false;
          break;
        }
        const int h = np_split(n);
        if ((q >> t) & 1) {
          lo += h;
          n -= h;
        } else {
          n = h;
        }
      }
      const int vi = cnt - 1 + q;
      s.kind[vi] = !exists ? 0 : (n <= kNpLeaf ? 1 : 2);
      if (exists && n <= kNpLeaf) {
        const int k = atomicAdd(&s.nleaf, 1);
        s.leaf_lo[k] = (int16_t)lo;
        s.leaf_n[k] = (int16_t)n;
        s.leaf_v[k] = (int16_t)vi;
      }
    }
  }
  __syncthreads();
  // B: leaves, 8 lanes each (lane k = accumulator r[k], its <= 16 loads in
  // flight before the serial adds), combined by xor shuffles 1, 2, 4
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane & 7;
    const int nw = blockDim.x >> 5, nleaf = s.nleaf;
    for (int L0 = warp * 4; L0 < nleaf; L0 += nw * 4) {
      const int L = L0 + (lane >> 3);
      const bool act = L < nleaf;
      const double v = np_leaf8(src, act ? s.leaf_lo[L] : 0, act ? s.leaf_n[L] : 0, sub);
      if (act && sub == 0) s.V[s.leaf_v[L]] = v;
    }
  }
  __syncthreads();
  // C: internal nodes bottom-up
  for (int r = kNpDepth - 1; r >= 0; --r) {
    const int cnt = 1 << r;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
      const int vi = cnt - 1 + q;
      if (s.kind[vi] == 2) s.V[vi] = __dadd_rn(s.V[2 * vi + 1], s.V[2 * vi + 2]);
    }
    __syncthreads();
  }
  return s.V[0];
}

}  // namespace fk

// One empty kernel per translation unit: its address identifies the unit's
// CUDA module, so fk_preload() can load every function of the module up front
// (lazy module loading would otherwise load each kernel at its first launch).
#define FK_MODULE_ANCHOR(name)                     \
  __global__ void k_module_anchor_##name() {}      \
  const void* module_anchor_##name() { return (const void*)k_module_anchor_##name; }

