// AUTX_ORDER_RADIX: the literal "stable priority sort" of SURVEY §8(a) row a5 — every active
// call gets a packed 64-bit key
//     q:4 | (arrival - arr_base):27 | not-running:1 | seq:32          (R11, R12; seq = row)
// and the keys are sorted by a stable LSD radix sort, one byte per digit.  The table is kept in
// seq (row) order, so sorting the high 32 bits stably already orders the low 32: only digits
// 4..7 are sorted, and a digit whose 256-bin histogram is a single bin (all keys equal there)
// is skipped.  The first min(BS, n_live) sorted keys become finalize's candidate list, and
// finalize cuts the prefix exactly as in the selection path, so both modes give identical
// decisions (tests/test_parity_gpu.py::test_radix_equals_select).
//
//   k_keys     dense pass: anti-starvation (same arithmetic as k_scan) + key pack + the four
//              global 256-bin digit histograms (for skip detection)
//   k_hist     per-tile 256-bin histogram of one digit        -> hist[digit value][tile]
//   k_scan_h   exclusive scan of hist in (digit value, tile) order (one CTA)
//   k_scatter  stable per-tile ranking (warp match + per-warp running counters) and scatter
//   k_take     the first min(BS, n_live) keys -> candidate rows
#include "autx_internal.cuh"
#include "block_prims.cuh"
#include "../../include/autx.h"

namespace autx {

constexpr int RX_THREADS = 256;
constexpr int RX_ITEMS = 16;                      // keys per thread
constexpr int RX_TILE = RX_THREADS * RX_ITEMS;   // 4096 keys per tile
constexpr int RX_WARP_KEYS = 32 * RX_ITEMS;      // 512 keys per warp, contiguous

__global__ void __launch_bounds__(RX_THREADS) k_keys(Policy pol, CallTable ct, ProgTable pt, Ctl* ctl,
                                                     RadixState rx, uint32_t t, uint32_t n_rows,
                                                     uint32_t arr_base) {
  __shared__ uint32_t h[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += RX_THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
  uint32_t npromo = 0, nlive = 0;
  const uint32_t n_pad = (n_rows + RX_TILE - 1) / RX_TILE * RX_TILE;
  for (uint32_t r = blockIdx.x * RX_THREADS + threadIdx.x; r < n_pad; r += gridDim.x * RX_THREADS) {
    uint64_t key = ~0ull;
    if (r < n_rows) {
      uint32_t qf = ct.qf[r];
      if (!(qf & QF_DEAD)) {
        ++nlive;
        uint32_t q = qf & QF_QMASK;
        if (pol.beta_den != 0) {
          uint32_t p = ct.prog[r], b = ct.base[r], m = ct.mtime[r];
          const PInfo pi = pt.info[p];
          uint64_t W = pi.pwait + (uint64_t)(t - b - m);
          uint64_t T = (uint64_t)pi.svc + m;
          if (!(W == 0 && T == 0) && mul_ge(W, pol.beta_den, T, pol.beta_num)) {  // Alg. 1 l.26
            q = 0;
            ct.qf[r] = (uint8_t)(qf & ~QF_QMASK);
            ct.base[r] = t;
            ct.mtime[r] = 0;
            ct.quanta[r] = pol.quanta[0];
            ++npromo;
          }
        }
        uint64_t arel = (uint64_t)(ct.arr[r] - arr_base) & ((1u << 27) - 1);
        key = ((uint64_t)q << 60) | (arel << 33) | ((uint64_t)((qf & QF_RUN) ? 0u : 1u) << 32) | r;
      }
    }
    if (r < n_pad) rx.keys[r] = key;
#pragma unroll
    for (int d = 0; d < 4; ++d) atomicAdd(&h[d][(uint32_t)(key >> (32 + 8 * d)) & 0xffu], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 256; i += RX_THREADS) {
    uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(&rx.dig_hist[i], v);
  }
  npromo = warp_sum(npromo);
  nlive = warp_sum(nlive);
  if (lane_id() == 0) {
    if (npromo) atomicAdd(&ctl->n_promoted, npromo);
    if (nlive) atomicAdd(&ctl->n_live, nlive);
  }
}

__global__ void __launch_bounds__(RX_THREADS) k_hist(const uint64_t* keys, uint32_t* hist, uint32_t ntiles,
                                                     int shift) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t* k = keys + (size_t)blockIdx.x * RX_TILE;
#pragma unroll 4
  for (int i = 0; i < RX_ITEMS; ++i) {
    uint64_t key = k[i * RX_THREADS + threadIdx.x];
    atomicAdd(&h[(uint32_t)(key >> shift) & 0xffu], 1u);
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan over 256 * ntiles counters in (digit, tile) order, one CTA of 1024 threads
__global__ void __launch_bounds__(1024) k_scan_h(uint32_t* hist, uint32_t n) {
  __shared__ uint32_t red[33];
  uint32_t per = (n + 1023) / 1024;
  uint32_t a = threadIdx.x * per, b = min(n, a + per);
  uint32_t s = 0;
  for (uint32_t i = a; i < b; ++i) s += hist[i];
  uint32_t off = block_excl_scan<uint32_t, 1024>(s, red, nullptr);
  for (uint32_t i = a; i < b; ++i) {
    uint32_t v = hist[i];
    hist[i] = off;
    off += v;
  }
}

// Stable scatter of one digit.  Warp w of a tile owns keys [w*512, (w+1)*512) of the tile in
// order; pass 1 counts its digits, a per-bin exclusive scan across warps gives each warp's base,
// pass 2 walks the 512 keys in order (32 at a time) ranking equal digits with __match_any_sync.
__global__ void __launch_bounds__(RX_THREADS) k_scatter(const uint64_t* in, uint64_t* out,
                                                        const uint32_t* hist, uint32_t ntiles,
                                                        int shift) {
  __shared__ uint32_t wh[RX_THREADS / 32][256];
  __shared__ uint32_t gbase[256];
  const uint32_t w = warp_id(), lane = lane_id();
  for (int i = lane; i < 256; i += 32) wh[w][i] = 0;
  const uint64_t* k = in + (size_t)blockIdx.x * RX_TILE + w * RX_WARP_KEYS;
  uint64_t key[RX_ITEMS];
#pragma unroll
  for (int i = 0; i < RX_ITEMS; ++i) key[i] = k[i * 32 + lane];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < RX_ITEMS; ++i) {
    uint32_t d = (uint32_t)(key[i] >> shift) & 0xffu;
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (lane == (uint32_t)(__ffs(peers) - 1)) wh[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per bin: exclusive scan across warps; global base of this tile's bin
  {
    uint32_t d = threadIdx.x;  // 256 threads == 256 bins
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < RX_THREADS / 32; ++ww) {
      uint32_t v = wh[ww][d];
      wh[ww][d] = run;
      run += v;
    }
    gbase[d] = hist[(size_t)d * ntiles + blockIdx.x];
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1;
#pragma unroll
  for (int i = 0; i < RX_ITEMS; ++i) {
    uint32_t d = (uint32_t)(key[i] >> shift) & 0xffu;
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t rank = wh[w][d] + __popc(peers & lt);
    out[gbase[d] + rank] = key[i];
    __syncwarp();
    if (lane == (uint32_t)(__ffs(peers) - 1)) wh[w][d] += __popc(peers);
    __syncwarp();
  }
}

__global__ void k_take(const uint64_t* keys, CallTable ct, Ctl* ctl, Outputs out, uint32_t BS, uint32_t K,
                       uint32_t t) {
  uint32_t n = min(BS, ctl->n_live);
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    uint32_t sl = (uint32_t)keys[i];
    CandRec r;
    load_rec(ct, sl, &r);
    out.cand[i] = sl;
    out.cand_rec[i] = r;
    out.ckey[i] = cand_key(r, t);
  }
  // previous batch: records for preempt; no region B (the full sort already ranked them)
  for (uint32_t j = threadIdx.x; j < ctl->n_prev; j += blockDim.x) {
    load_rec(ct, out.prev_slots[j], out.prev_rec + j);
    out.ckey[n + j] = ~0ull;
  }
  if (threadIdx.x == 0) {
    ctl->n_cand_a = n;
    ctl->n_cand_b = 0;
    ctl->qstar = K;  // no extra running candidates: the sort already ordered them
  }
}

cudaError_t launch_radix_order(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl,
                               Outputs out, RadixState rx, uint32_t t, uint32_t n_rows,
                               uint32_t arr_base, int sms, uint32_t* passes_out) {
  const uint32_t ntiles = std::max<uint32_t>(1, (n_rows + RX_TILE - 1) / RX_TILE);
  const uint32_t n_pad = ntiles * RX_TILE;
  cudaMemsetAsync(rx.dig_hist, 0, 4 * 256 * sizeof(uint32_t), s);
  uint32_t grid = std::min<uint32_t>(ntiles * RX_ITEMS, (uint32_t)sms * 8);
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_keys<<<grid, RX_THREADS, 0, s>>>(pol, ct, pt, ctl, rx, t, n_rows, arr_base);
  // skip detection needs the digit histograms on the host (a 4 KB read; this mode is the
  // contract path, the selection path is the fast path)
  cudaMemcpyAsync(rx.h_dig_hist, rx.dig_hist, 4 * 256 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  uint64_t* a = rx.keys;
  uint64_t* b = rx.keys_alt;
  uint32_t passes = 0;
  for (int d = 0; d < 4; ++d) {
    bool uniform = false;
    for (int v = 0; v < 256; ++v)
      if (rx.h_dig_hist[d * 256 + v] == n_pad) uniform = true;
    if (uniform) continue;
    int shift = 32 + 8 * d;
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
    k_hist<<<ntiles, RX_THREADS, 0, s>>>(a, rx.tile_hist, ntiles, shift);
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
    k_scan_h<<<1, 1024, 0, s>>>(rx.tile_hist, 256 * ntiles);
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
    k_scatter<<<ntiles, RX_THREADS, 0, s>>>(a, b, rx.tile_hist, ntiles, shift);
    std::swap(a, b);
    ++passes;
  }
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_take<<<1, 1024, 0, s>>>(a, ct, ctl, out, pol.max_batch, pol.K, t);
  if (passes_out) *passes_out = passes;
  return cudaGetLastError();
}

}  // namespace autx
