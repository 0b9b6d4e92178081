// Microbenchmark: single-CTA sort of 2048 (u64 key, u32 payload) pairs, 1024 threads.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include "../../paper_2502_13965_b200/csrc/block_prims.cuh"
using namespace autx;

extern __shared__ unsigned char dsm[];
__global__ void __launch_bounds__(1024) k_sort(const uint64_t* in, uint64_t* out, long long* cyc, int mode, int reps) {
  uint64_t* khi = (uint64_t*)dsm;
  uint64_t* k2 = khi + 2048;
  uint32_t* klo = (uint32_t*)(k2 + 2048);
  uint32_t* p2 = klo + 2048;
  const uint32_t tid = threadIdx.x;
  long long total = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (uint32_t i = tid; i < 2048; i += 1024) { khi[i] = in[i]; klo[i] = i; }
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) {
      bitonic_sort_pairs<1024>(khi, klo, 2048);
    } else if (mode == 2) {
      block_merge_sort<1024>(khi, klo, k2, p2);
    } else {
      uint64_t k0 = khi[2 * tid], k1 = khi[2 * tid + 1];
      uint32_t v0 = klo[2 * tid], v1 = klo[2 * tid + 1];
      __syncthreads();
      bitonic_sort_reg2<1024>(k0, v0, k1, v1, khi, klo);
      khi[2 * tid] = k0; klo[2 * tid] = v0; khi[2 * tid + 1] = k1; klo[2 * tid + 1] = v1;
      __syncthreads();
    }
    long long t1 = clock64();
    total += t1 - t0;
  }
  for (uint32_t i = tid; i < 2048; i += 1024) out[i] = khi[i];
  if (tid == 0) *cyc = total / reps;
}

int main() {
  std::vector<uint64_t> h(2048);
  uint64_t x = 88172645463325252ull;
  for (auto& v : h) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = x >> 1; }
  uint64_t *din, *dout; long long* dc;
  cudaMalloc(&din, 2048 * 8); cudaMalloc(&dout, 2048 * 8); cudaMalloc(&dc, 8);
  cudaMemcpy(din, h.data(), 2048 * 8, cudaMemcpyHostToDevice);
  auto ref = h; std::sort(ref.begin(), ref.end());
  cudaFuncSetAttribute(k_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int mode = 0; mode < 3; ++mode) {
    k_sort<<<1, 1024, 48 * 1024>>>(din, dout, dc, mode, 20);
    cudaDeviceSynchronize();
    long long c; std::vector<uint64_t> o(2048);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(o.data(), dout, 2048 * 8, cudaMemcpyDeviceToHost);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k_sort<<<1, 1024, 48 * 1024>>>(din, dout, dc, mode, 1); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("mode %d (%s): %lld cycles per sort (%.2f us at 1.9 GHz), single-launch kernel %.2f us, correct=%d\n", mode,
           mode == 2 ? "merge" : mode ? "reg/shuffle" : "smem", c, c / 1900.0, ms * 1e3, (int)(o == ref));
  }
  return 0;
}
