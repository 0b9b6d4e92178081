// Instruction-fetch cost of straight-line code run once by one CTA (cold vs warm), B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ifetch ifetch.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
template <int N>
__device__ __forceinline__ unsigned body(unsigned x, unsigned k, unsigned c) {
  unsigned a = x, b = x + 1, e = x + 2, d = x + 3;  // 4 independent chains: issue-bound, not latency-bound
#pragma unroll
  for (int i = 0; i < N; i += 4) {
    a = a * k + c; b = b * k + c; e = e * k + c; d = d * k + c;
    k ^= a; c += d;  // keep the chains opaque
  }
  return a ^ b ^ e ^ d;
}
// pass 0 cold, pass 1 warm (same code), then a second cold region of the same size
template <int N>
__global__ void k(unsigned* out, unsigned long long* ts, const unsigned* kc) {
  unsigned x = threadIdx.x;
  for (int pass = 0; pass < 2; ++pass) {
    __syncthreads();
    unsigned long long t0 = gt();
    x = body<N>(x, kc[0], kc[1]);
    __syncthreads();
    if (threadIdx.x == 0) ts[pass] = gt() - t0;
  }
  out[threadIdx.x] = x;
}
int main() {
  unsigned* o; unsigned long long* ts; cudaMalloc(&o, 4096); cudaMallocManaged(&ts, 64);
  void* flush; size_t fb = 512u << 20; cudaMalloc(&flush, fb);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(flush, rep, fb);
    k<2048><<<1, 32>>>(o, ts, o); cudaDeviceSynchronize();
    printf("2048 instr (32 KB): cold %.2f us  warm %.2f us\n", ts[0] / 1e3, ts[1] / 1e3);
    cudaMemset(flush, rep, fb);
    k<8192><<<1, 32>>>(o, ts, o); cudaDeviceSynchronize();
    printf("8192 instr (128 KB): cold %.2f us  warm %.2f us\n", ts[0] / 1e3, ts[1] / 1e3);
    k<8192><<<1, 32>>>(o, ts, o); cudaDeviceSynchronize();
    printf("8192 instr, no flush: first %.2f us  second %.2f us\n", ts[0] / 1e3, ts[1] / 1e3);
  }
  return 0;
}
