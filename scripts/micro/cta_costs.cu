// Cost model of single-CTA phases on B200: block scan (512 thr), __syncthreads, dependent L2 /
// DRAM round trips, coalesced 48 KB L2 read.  One CTA, %globaltimer and clock64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cta_costs_bin cta_costs.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2502_13965_b200/csrc/block_prims.cuh"
using namespace autx;

__global__ void k(uint32_t* chain, const uint4* big, unsigned long long* out, int reps) {
  __shared__ unsigned long long red[33];
  uint32_t tid = threadIdx.x;
  // (a) block scans
  __syncthreads();
  long long c0 = clock64();
  unsigned long long acc = tid;
  for (int i = 0; i < reps; ++i) acc = block_excl_scan<unsigned long long, 512>(acc + 1, red, nullptr);
  long long c1 = clock64();
  // (b) bare __syncthreads
  for (int i = 0; i < reps; ++i) __syncthreads();
  long long c2 = clock64();
  // (c) dependent L2-resident pointer chase (thread 0)
  uint32_t p = 0;
  if (tid == 0) for (int i = 0; i < reps; ++i) p = __ldcg(chain + p);
  __syncthreads();
  long long c3 = clock64();
  // (d) coalesced 48 KB read by 512 threads (L2-resident), 6 uint4 per thread, one round
  uint4 s = make_uint4(0, 0, 0, 0);
  for (int r = 0; r < 6; ++r) { uint4 v = __ldcg(big + r * 512 + tid); s.x ^= v.x; s.y ^= v.y; }
  __syncthreads();
  long long c4 = clock64();
  if (tid == 0) {
    out[0] = (c1 - c0) / reps; out[1] = (c2 - c1) / reps; out[2] = (c3 - c2) / reps; out[3] = c4 - c3;
    out[4] = acc + p + s.x + s.y;
  }
}

int main() {
  uint32_t* chain; uint4* big; unsigned long long* out;
  const int N = 1 << 20;
  cudaMalloc(&chain, N * 4); cudaMalloc(&big, 1 << 20); cudaMallocManaged(&out, 64);
  uint32_t* h = new uint32_t[N];
  for (int i = 0; i < N; ++i) h[i] = (uint32_t)((i * 2654435761u + 12345u) % N);  // random chain
  cudaMemcpy(chain, h, N * 4, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    k<<<1, 512>>>(chain, big, out, 64);   // warm
    k<<<1, 512>>>(chain, big, out, 64);
    cudaDeviceSynchronize();
    printf("cycles: block_excl_scan<u64,512> %llu | __syncthreads %llu | dependent L2 load %llu | 48KB coalesced L2 read %llu\n",
           out[0], out[1], out[2], out[3]);
  }
  // DRAM: a fresh chain region each time (cold)
  void* fl; cudaMalloc(&fl, 512u << 20);
  cudaMemset(fl, 1, 512u << 20);
  k<<<1, 512>>>(chain, big, out, 64);
  cudaDeviceSynchronize();
  printf("after L2 flush: dependent load %llu cycles (mostly DRAM), 48KB read %llu\n", out[2], out[3]);
  return 0;
}
