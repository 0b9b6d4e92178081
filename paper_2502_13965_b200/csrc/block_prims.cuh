// Warp/block primitives (scans, reductions, 128-bit compare, PDL, timers) written for sm_100a.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace autx {

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane_id() >= (uint32_t)d) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Block-wide exclusive scan; every thread of the block must call it.  smem: >= 33 T.
template <typename T, int NT>
__device__ __forceinline__ T block_excl_scan(T v, T* smem, T* total) {
  constexpr int NW = NT / 32;
  T inc = warp_incl_scan(v);
  if (lane_id() == 31) smem[warp_id()] = inc;
  __syncthreads();
  if (warp_id() == 0) {
    T w = lane_id() < NW ? smem[lane_id()] : T(0);
    T wi = warp_incl_scan(w);
    if (lane_id() < NW) smem[lane_id()] = wi - w;
    if (lane_id() == NW - 1) smem[32] = wi;
  }
  __syncthreads();
  T r = smem[warp_id()] + inc - v;
  if (total) *total = smem[32];
  __syncthreads();
  return r;
}

// 128-bit compare: a*b >= c*d for u64 a, c and u32 b, d.
__device__ __forceinline__ bool mul_ge(uint64_t a, uint32_t b, uint64_t c, uint32_t d) {
  if (((a | c) >> 32) == 0) return a * (uint64_t)b >= c * (uint64_t)d;  // both products < 2^64
  uint64_t l1 = a * (uint64_t)b, h1 = __umul64hi(a, (uint64_t)b);
  uint64_t l2 = c * (uint64_t)d, h2 = __umul64hi(c, (uint64_t)d);
  return h1 > h2 || (h1 == h2 && l1 >= l2);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start before its predecessor ends;
// pdl_wait() blocks until the predecessor grid completed and its writes are visible, and
// pdl_trigger() lets the successor launch as soon as every CTA of this grid has started.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Bounds checks of a debug build (AUTX_NVCC_FLAGS=-DAUTX_BOUNDS): print the site and trap.  The
// pool refuses compute-sanitizer, so out-of-bounds indices are caught by these instead.
#ifdef AUTX_BOUNDS
#define AUTX_CHECK(cond, what, v)                                                                        \
  do {                                                                                                  \
    if (!(cond)) {                                                                                      \
      printf("AUTX_CHECK failed: %s (%s:%d) value %llu block %d thread %d\n", what, __FILE__, __LINE__, \
             (unsigned long long)(v), (int)blockIdx.x, (int)threadIdx.x);                               \
      __trap();                                                                                         \
    }                                                                                                   \
  } while (0)
#else
#define AUTX_CHECK(cond, what, v) do { } while (0)
#endif

__device__ __forceinline__ uint32_t ceil_div_u32(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

}  // namespace autx
