// Probe: tcgen05.ld (TMEM -> registers) throughput per SM on B200, the
// resource the FlashAssign epilogue spends most of its time in (it must read
// every N x K fp32 distance out of TMEM once: 137 GB per config-3 iteration).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_09229_b200/csrc
//        scripts/probe_tmem_ld.cu -o /tmp/probe_ld
#include <cstdio>
#include <cstdint>
#include "fk_common.cuh"

using namespace fk;

template <int DEPTH>
__global__ void __launch_bounds__(512, 1) probe(int reps, int nwarps, unsigned long long* cyc, float* sink) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = holder;
  float acc = 0.f;
  unsigned long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t q = warp & 3;
    const uint32_t col0 = (warp >> 2) * 32;
    uint32_t v[DEPTH][32];
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < DEPTH; ++k) {
        const uint32_t col = (col0 + (r * DEPTH + k) * 128) & 511;
        FK_TMEM_LD_32x32b_X32(tb + (q * 32 << 16) + col, v[k]);
      }
#pragma unroll
      for (int k = 0; k < DEPTH; ++k) {
        FK_TMEM_WAIT_LD(v[k]);
        acc += __uint_as_float(v[k][0]) + __uint_as_float(v[k][31]);
      }
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, sms * 8);
  cudaMalloc(&sink, sms * 512 * 4);
  const int reps = 4000;
  for (int nw : {4, 8, 12, 16}) {
    for (int depth : {1, 2, 4}) {
      auto run = [&]() {
        if (depth == 1) probe<1><<<sms, 512>>>(reps, nw, cyc, sink);
        else if (depth == 2) probe<2><<<sms, 512>>>(reps / 2, nw, cyc, sink);
        else probe<4><<<sms, 512>>>(reps / 4, nw, cyc, sink);
      };
      run();
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      unsigned long long c0 = 0;
      cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes_sm = (double)nw * reps * 32 * 32 * 4;  // per SM
      printf("warps=%2d depth=%d: %.1f B/clk/SM (clock64), %.2f TB/s aggregate (events), err=%s\n", nw,
             depth, bytes_sm / c0, bytes_sm * sms / (ms * 1e-3) / 1e12,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
