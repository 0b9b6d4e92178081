// Does one CTA's L2 access slow down right after a grid-wide read/write burst + grid barrier?
// 246 CTAs x 512 threads: tiles read 56 KB and write 16 KB each, fence, arrive; the last CTA
// waits, then times a coalesced 48 KB read of data CTA 0 wrote and a block scan (clock64).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2502_13965_b200/csrc/block_prims.cuh"
using namespace autx;

__global__ void __launch_bounds__(512, 2) k(const uint4* in, uint4* wr, uint4* xrec, unsigned* bar,
                                            unsigned long long* out, int burst) {
  __shared__ unsigned long long red[33];
  const uint32_t tid = threadIdx.x;
  const uint32_t fin = gridDim.x - 1;
  if (blockIdx.x != fin) {
    if (burst) {
      uint4 acc = make_uint4(0, 0, 0, 0);
      const uint4* src = in + (size_t)blockIdx.x * 3584;
      for (int r = 0; r < 7; ++r) { uint4 v = __ldcs(src + r * 512 + tid); acc.x ^= v.x; acc.y += v.y; }
      wr[(size_t)blockIdx.x * 1024 + tid] = acc;
      wr[(size_t)blockIdx.x * 1024 + 512 + tid] = acc;
    }
    if (blockIdx.x == 0) {
      if (burst < 2) {
        for (int r = 0; r < 6; ++r) xrec[r * 512 + tid] = make_uint4(tid, r, 1, 2);
      } else {
        // like the extraction: 48-B records, thread t writes records 8t' .. (rows of one thread),
        // 3 x 16 B each, lanes 8 records apart (scattered partial sectors)
        for (int k = 0; k < 2; ++k) {
          const uint32_t rec = (tid % 128) * 8 + (tid / 128) * 2 + k;  // 1024 records
          uint4* d = xrec + rec * 3;
          d[0] = make_uint4(rec, 1, 2, 3); d[1] = make_uint4(4, 5, 6, 7); d[2] = make_uint4(8, 0, 0, 0);
        }
      }
    }
    __syncthreads();
    if (tid == 0) { __threadfence(); atomicAdd(bar, 1u); }
    return;
  }
  if (tid == 0) { while (atomicAdd(bar, 0u) < gridDim.x - 1) __nanosleep(20); }
  __syncthreads();
  long long c0 = clock64();
  uint4 s = make_uint4(0, 0, 0, 0);
  for (int r = 0; r < 6; ++r) { uint4 v = __ldcg(xrec + r * 512 + tid); s.x ^= v.x; s.y += v.y; }
  __syncthreads();
  long long c1 = clock64();
  unsigned long long a = s.x;
  for (int i = 0; i < 8; ++i) a = block_excl_scan<unsigned long long, 512>(a + 1, red, nullptr);
  long long c2 = clock64();
  if (tid == 0) { out[0] = c1 - c0; out[1] = (c2 - c1) / 8; out[2] = a + s.y; *bar = 0; }
}

int main() {
  uint4 *in, *wr, *xrec; unsigned* bar; unsigned long long* out;
  cudaMalloc(&in, 246ull * 3584 * 16); cudaMalloc(&wr, 246ull * 1024 * 16); cudaMalloc(&xrec, 6 * 512 * 16);
  cudaMalloc(&bar, 4); cudaMemset(bar, 0, 4); cudaMallocManaged(&out, 64);
  void* fl; cudaMalloc(&fl, 512u << 20);
  for (int burst = 0; burst < 3; ++burst)
    for (int flush = 0; flush < 2; ++flush)
      for (int rep = 0; rep < 3; ++rep) {
        if (flush) cudaMemset(fl, rep, 512u << 20);
        k<<<246, 512>>>(in, wr, xrec, bar, out, burst);
        cudaDeviceSynchronize();
        if (rep == 2) printf("burst=%d flush=%d: 48KB read after barrier %llu cyc, u64 block scan %llu cyc\n", burst, flush, out[0], out[1]);
      }
  return 0;
}
