// Microbenchmark: match.any.sync latency/throughput vs distinct values per warp,
// ballot-based match, and shared atomics with intra-warp address conflicts.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_match scripts/probe_match.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_match(int iters, int distinct, unsigned* out, int dep) {
  unsigned acc = 0;
  unsigned v = (threadIdx.x & 31) % distinct;
  for (int i = 0; i < iters; ++i) {
    unsigned m = __match_any_sync(0xffffffffu, v + (dep ? (acc & 1) : 0) * 0);
    acc += m;
    if (dep) v = (v + (m & 1)) % 4096 + ((threadIdx.x & 31) % distinct) * 4096;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_ballot(int iters, int distinct, unsigned* out) {
  unsigned acc = 0;
  unsigned v = (threadIdx.x & 31) % distinct;
  for (int i = 0; i < iters; ++i) {
    unsigned m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 12; ++b) {
      const bool bit = (v >> b) & 1;
      const unsigned bal = __ballot_sync(0xffffffffu, bit);
      m &= bit ? bal : ~bal;
    }
    acc += m;
    v = (v + (m & 1)) & 4095;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_atoms(int iters, int distinct, unsigned* out) {
  __shared__ unsigned sh[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const unsigned w = threadIdx.x >> 5;
  unsigned v = ((threadIdx.x & 31) % distinct) * 2 + w * 64;
  for (int i = 0; i < iters; ++i) atomicAdd(&sh[(v + i * 7) & 4095], 1u);
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sh[threadIdx.x];
}

int main() {
  unsigned* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (int kind = 0; kind < 4; ++kind)
    for (int distinct : {1, 2, 8, 32}) {
      for (int warps : {1, 32}) {
        const int blocks = 148, threads = 32 * warps;
        auto launch = [&]() {
          if (kind == 0) k_match<<<blocks, threads>>>(iters, distinct, out, 0);
          if (kind == 1) k_match<<<blocks, threads>>>(iters, distinct, out, 1);
          if (kind == 2) k_ballot<<<blocks, threads>>>(iters, distinct, out);
          if (kind == 3) k_atoms<<<blocks, threads>>>(iters, distinct, out);
        };
        launch();
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double cyc = ms * 1e-3 * 1.9e9 / iters;  // cycles per iteration (approx clock)
        const char* names[] = {"match indep", "match dep", "ballot12 dep", "atoms"};
        printf("%-13s distinct=%2d warps/SM=%2d: %7.1f cycles/iter per warp, %6.2f iters/cycle/SM\n",
               names[kind], distinct, warps, cyc, warps / cyc);
      }
    }
  return 0;
}
