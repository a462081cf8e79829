// Probe: how tcgen05.cp (smem -> TMEM) maps a no-swizzle matrix descriptor
// onto TMEM lanes/columns, including stride-0 row groups (broadcast), for
// cta_group::1 and cta_group::2.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -I paper_2603_09229_b200/csrc scripts/probe_tmem_cp.cu -o /tmp/probe_cp
#include <cstdio>
#include <cstdint>
#include <vector>
#include "fk_common.cuh"

using namespace fk;

constexpr int NV = 6;

__device__ uint64_t desc_none(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46);
}

template <int CG>
__global__ void __cluster_dims__(2, 1, 1) probe(float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* src = reinterpret_cast<float*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8192);
  uint32_t* holder = reinterpret_cast<uint32_t*>(smem + 8192 + 64);
  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) src[i] = float(rank * 100000 + i);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (CG == 2) tmem_alloc_cg2<256>(holder); else tmem_alloc<256>(holder);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tb = *holder;
  const uint32_t a = smem_u32(src);
  if (warp == 0 && (CG == 1 || rank == 0) && elect_one()) {
    // v0: 128x256b LBO=128 SBO=256 (distinct rows);  v1: 128x256b LBO=128 SBO=0
    // v2: 128x256b LBO=256 SBO=128;                  v3: 32x128b.warpx4 SBO=128
    // v4: 32x128b.warpx4 SBO=0;                      v5: 128x256b LBO=128 SBO=0 start +512
    uint64_t d[NV] = {desc_none(a, 128, 256), desc_none(a, 128, 0), desc_none(a, 256, 128),
                      desc_none(a, 128, 128), desc_none(a, 128, 0), desc_none(a + 512, 128, 0)};
    if (CG == 2) {
      asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(tb + 0), "l"(d[0]));
      asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(tb + 8), "l"(d[1]));
      asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(tb + 16), "l"(d[2]));
      asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(tb + 24), "l"(d[3]));
      asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(tb + 32), "l"(d[4]));
      asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(tb + 40), "l"(d[5]));
      tc_commit_cg2_mc(bar, 0x3);
    } else {
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tb + 0), "l"(d[0]));
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tb + 8), "l"(d[1]));
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tb + 16), "l"(d[2]));
      asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tb + 24), "l"(d[3]));
      asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tb + 32), "l"(d[4]));
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tb + 40), "l"(d[5]));
      tc_commit(bar);
    }
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc_fence_after();
  if (warp < 4) {
    uint32_t v[32];
    for (int base = 0; base < 64; base += 32) {
      FK_TMEM_LD_32x32b_X32(tb + (uint32_t(warp * 32) << 16) + base, v);
      FK_TMEM_WAIT_LD(v);
      for (int j = 0; j < 32; ++j)
        out[((size_t)rank * 128 + warp * 32 + lane) * 64 + base + j] = __uint_as_float(v[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_cg2<256>(tb); else tmem_dealloc<256>(tb);
  }
}

template <int CG>
static void run() {
  float* d;
  cudaMalloc(&d, 2 * 128 * 64 * 4);
  cudaMemset(d, 0xff, 2 * 128 * 64 * 4);
  cudaFuncSetAttribute(probe<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 9216);
  probe<CG><<<2, 128, 9216>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("== cta_group::%d: %s\n", CG, cudaGetErrorString(e));
  std::vector<float> h(2 * 128 * 64);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  const char* names[NV] = {"128x256b L128 S256", "128x256b L128 S0", "128x256b L256 S128",
                           "32x128b.w4 S128", "32x128b.w4 S0", "128x256b L128 S0 +512B"};
  for (int v = 0; v < NV; ++v) {
    const int w = (v == 3 || v == 4) ? 4 : 8;
    printf("-- %s\n", names[v]);
    for (int r = 0; r < 2; ++r)
      for (int lane : {0, 1, 2, 7, 8, 9, 15, 16, 31, 32, 33, 63, 64, 127}) {
        printf("rank %d lane %3d:", r, lane);
        for (int c = 0; c < w; ++c) printf(" %7.0f", h[((size_t)r * 128 + lane) * 64 + v * 8 + c]);
        printf("\n");
      }
  }
  cudaFree(d);
}

int main() {
  run<1>();
  run<2>();
  return 0;
}
