// sm_100a paged KV swap.
//
// A preempted call's KV lives in per-layer paged pools: for layer l, K|V, GPU block b the chunk
// pool[l][kv] + b * chunk_bytes.  Its host copy is ONE contiguous range of the pinned arena laid
// out [block j][layer l][K|V][chunk] ("consolidate all KV blocks into a single contiguous
// chunk").  The work unit is one (plan block, layer, K|V) chunk.
//
//   k_swap_sm      SM-driven copy straight between HBM and the mapped pinned arena (posted
//                  16-B stores over PCIe for swap-out, 16-B loads with deep MLP for swap-in).
//   k_stage        gather (swap-out) / scatter (swap-in) between the paged pool and a
//                  contiguous device staging buffer, for the copy-engine DMA variant (the
//                  paper's own scheme: gather, then one bulk transfer per call).
#include "autx_internal.cuh"

namespace autx {

struct SwapGeom {
  uint32_t n_layers;
  uint32_t chunk_bytes;
  uint64_t page_bytes;  // n_layers * 2 * chunk_bytes
};

__device__ __forceinline__ uint32_t find_item(const PlanItem* items, uint32_t n, uint32_t b) {
  // largest i with items[i].blk_off <= b (blk_off ascending)
  uint32_t lo = 0, hi = n;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (items[mid].blk_off <= b) lo = mid; else hi = mid;
  }
  return lo;
}

template <int UNROLL>
__device__ __forceinline__ void copy_chunk(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                           uint32_t n16) {
  for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x * UNROLL) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      uint32_t k = i + u * blockDim.x;
      if (k < n16) v[u] = __ldcs(src + k);  // streamed: do not pollute L2
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      uint32_t k = i + u * blockDim.x;
      if (k < n16) __stcs(dst + k, v[u]);
    }
  }
}

// direction 0: swap-out (pool -> host arena); 1: swap-in (host arena -> pool); 2: both at once
// (full duplex over the host link): even CTAs swap out, odd CTAs swap in
__global__ void __launch_bounds__(256) k_swap_sm(const Ctl* ctl, KvState kv, void* const* kpool,
                                                 void* const* vpool, SwapGeom g, char* arena,
                                                 int direction) {
  uint32_t cta = blockIdx.x, ncta = gridDim.x;
  if (direction == 2) {
    direction = (int)(blockIdx.x & 1u);
    cta = blockIdx.x >> 1;
    ncta = (gridDim.x + 1 - (uint32_t)direction) >> 1;
  }
  const uint32_t n_items = direction == 0 ? ctl->n_plan_out : ctl->n_plan_in;
  const uint32_t n_blocks = direction == 0 ? ctl->plan_out_chunks : ctl->plan_in_chunks;
  const PlanItem* items = direction == 0 ? kv.plan_out : kv.plan_in;
  const uint32_t* blocks = direction == 0 ? kv.plan_out_blocks : kv.plan_in_blocks;
  const uint64_t n_chunks = (uint64_t)n_blocks * g.n_layers * 2;
  const uint32_t n16 = g.chunk_bytes / 16;
  for (uint64_t c = cta; c < n_chunks; c += ncta) {
    uint32_t b = (uint32_t)(c / (2 * g.n_layers));
    uint32_t rem = (uint32_t)(c % (2 * g.n_layers));
    uint32_t l = rem >> 1, kvsel = rem & 1;
    uint32_t it = find_item(items, n_items, b);
    PlanItem item = items[it];
    uint32_t j = b - item.blk_off;
    char* pool = (char*)(kvsel ? vpool[l] : kpool[l]);
    uint4* dev = reinterpret_cast<uint4*>(pool + (uint64_t)blocks[b] * g.chunk_bytes);
    uint4* host = reinterpret_cast<uint4*>(arena + item.host_page * g.page_bytes +
                                           ((uint64_t)j * g.n_layers + l) * 2 * g.chunk_bytes +
                                           (uint64_t)kvsel * g.chunk_bytes);
    if (direction == 0) copy_chunk<8>(host, dev, n16);
    else copy_chunk<8>(dev, host, n16);
  }
}

// Staging layout: item i occupies [blk_off_i * page_bytes, (blk_off_i + nblk_i) * page_bytes),
// identical to its host range layout, so one cudaMemcpyAsync per call moves it.
__global__ void __launch_bounds__(256) k_stage(const Ctl* ctl, KvState kv, void* const* kpool,
                                               void* const* vpool, SwapGeom g, char* staging,
                                               int direction) {
  const uint32_t n_blocks = direction == 0 ? ctl->plan_out_chunks : ctl->plan_in_chunks;
  const uint32_t* blocks = direction == 0 ? kv.plan_out_blocks : kv.plan_in_blocks;
  const uint64_t n_chunks = (uint64_t)n_blocks * g.n_layers * 2;
  const uint32_t n16 = g.chunk_bytes / 16;
  for (uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    uint32_t b = (uint32_t)(c / (2 * g.n_layers));
    uint32_t rem = (uint32_t)(c % (2 * g.n_layers));
    uint32_t l = rem >> 1, kvsel = rem & 1;
    char* pool = (char*)(kvsel ? vpool[l] : kpool[l]);
    uint4* dev = reinterpret_cast<uint4*>(pool + (uint64_t)blocks[b] * g.chunk_bytes);
    uint4* st = reinterpret_cast<uint4*>(staging + (uint64_t)b * g.page_bytes +
                                         ((uint64_t)l * 2 + kvsel) * g.chunk_bytes);
    if (direction == 0) copy_chunk<8>(st, dev, n16);
    else copy_chunk<8>(dev, st, n16);
  }
}

cudaError_t launch_swap(cudaStream_t s, const Ctl* ctl, KvState kv, void* const* d_kpool,
                        void* const* d_vpool, uint32_t n_layers, uint32_t chunk_bytes,
                        char* host_arena, int direction, int n_ctas) {
  SwapGeom g{n_layers, chunk_bytes, (uint64_t)n_layers * 2 * chunk_bytes};
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_swap_sm<<<n_ctas, 256, 0, s>>>(ctl, kv, d_kpool, d_vpool, g, host_arena, direction);
  return cudaGetLastError();
}

cudaError_t launch_stage(cudaStream_t s, const Ctl* ctl, KvState kv, void* const* d_kpool,
                         void* const* d_vpool, uint32_t n_layers, uint32_t chunk_bytes,
                         char* staging, int direction, int n_ctas) {
  SwapGeom g{n_layers, chunk_bytes, (uint64_t)n_layers * 2 * chunk_bytes};
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_stage<<<n_ctas, 256, 0, s>>>(ctl, kv, d_kpool, d_vpool, g, staging, direction);
  return cudaGetLastError();
}

}  // namespace autx
