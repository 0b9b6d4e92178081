// AUTX_ORDER_RADIX: the literal "stable priority sort" of SURVEY §8(a) row a5 — every active
// call gets a packed 64-bit key
//     q:4 | (arrival - arr_base):27 | not-running:1 | seq:32          (R11, R12; seq = row)
// and the keys are sorted by a stable LSD radix sort, one byte per digit.  The table is kept in
// seq (row) order, so sorting the high 32 bits stably already orders the low 32: only digits
// 4..7 are sorted, and a digit whose 256-bin histogram is a single bin (all keys equal there)
// is skipped — decided on the device by every pass kernel from k_keys' global digit histograms,
// so the step needs no host round trip; a pass reads the key buffer the earlier non-skipped
// passes left (parity of their count).  The first min(BS, n_live) sorted keys become finalize's candidate list, and
// finalize cuts the prefix exactly as in the selection path, so both modes give identical
// decisions (tests/test_parity_gpu.py::test_radix_equals_select).
//
//   k_keys     dense pass: anti-starvation (same arithmetic as k_scan) + key pack + the four
//              global 256-bin digit histograms (for skip detection)
//   k_hist     per-tile 256-bin histogram of one digit        -> hist[digit value][tile]
//   k_scan_h   exclusive scan of hist in (digit value, tile) order: a warp per digit value scans
//              its tiles, the digit values' bases come from the global histogram
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

// Is digit d (of digits 4..7) a single bin over all n_pad keys (the pass is the identity)?  And
// which key buffer does pass d read (the number of earlier non-skipped passes, mod 2)?  Every
// CTA of a pass kernel derives both from the global digit histograms (block of >= 256 threads).
__device__ __forceinline__ bool digit_uniform(const uint32_t* dig_hist, int d, uint32_t n_pad) {
  const uint32_t v = threadIdx.x < 256 ? dig_hist[d * 256 + threadIdx.x] : 0u;
  return __syncthreads_or(v == n_pad) != 0;
}
__device__ __forceinline__ uint32_t pass_src(const uint32_t* dig_hist, int d, uint32_t n_pad) {
  uint32_t src = 0;
  for (int e = 0; e < d; ++e) src ^= digit_uniform(dig_hist, e, n_pad) ? 0u : 1u;
  return src;
}

__global__ void __launch_bounds__(RX_THREADS) k_hist(RadixState rx, uint32_t* hist, uint32_t ntiles, int d) {
  __shared__ uint32_t h[256];
  const uint32_t n_pad = ntiles * RX_TILE;
  if (digit_uniform(rx.dig_hist, d, n_pad)) return;
  const int shift = 32 + 8 * d;
  const uint64_t* keys = pass_src(rx.dig_hist, d, n_pad) ? rx.keys_alt : rx.keys;
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

// Exclusive scan of the (digit value, tile) counters: a warp per digit value walks its ntiles
// counters 32 at a time with a carry; the value's base is the exclusive prefix of the global
// digit histogram (k_keys) over the smaller values.  8 CTAs x 32 warps = the 256 values.
__global__ void __launch_bounds__(1024) k_scan_h(RadixState rx, uint32_t* hist, uint32_t ntiles, int d) {
  const uint32_t n_pad = ntiles * RX_TILE;
  if (digit_uniform(rx.dig_hist, d, n_pad)) return;
  const uint32_t v = blockIdx.x * 32 + warp_id(), lane = lane_id();
  // base of value v: sum of the global histogram over values < v (8 per lane)
  uint32_t b = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t u = lane * 8 + k;
    b += u < v ? rx.dig_hist[d * 256 + u] : 0u;
  }
  uint32_t carry = warp_sum(b);
  uint32_t* row = hist + (size_t)v * ntiles;
  for (uint32_t c0 = 0; c0 < ntiles; c0 += 32) {
    const uint32_t i = c0 + lane;
    const uint32_t x = i < ntiles ? row[i] : 0u;
    const uint32_t inc = warp_incl_scan(x);
    if (i < ntiles) row[i] = carry + inc - x;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
}

// Stable scatter of one digit.  Warp w of a tile owns keys [w*512, (w+1)*512) of the tile in
// order; pass 1 counts its digits, a per-bin exclusive scan across warps gives each warp's base,
// pass 2 walks the 512 keys in order (32 at a time) ranking equal digits with __match_any_sync.
__global__ void __launch_bounds__(RX_THREADS) k_scatter(RadixState rx, const uint32_t* hist, uint32_t ntiles,
                                                        int d) {
  __shared__ uint32_t wh[RX_THREADS / 32][256];
  __shared__ uint32_t gbase[256];
  const uint32_t n_pad = ntiles * RX_TILE;
  if (digit_uniform(rx.dig_hist, d, n_pad)) return;
  const int shift = 32 + 8 * d;
  const bool alt = pass_src(rx.dig_hist, d, n_pad) != 0;
  const uint64_t* in = alt ? rx.keys_alt : rx.keys;
  uint64_t* out = alt ? rx.keys : rx.keys_alt;
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

__global__ void __launch_bounds__(1024) k_take(RadixState rx, uint32_t n_pad, CallTable ct, Ctl* ctl, Outputs out,
                                               uint32_t BS, uint32_t K, uint32_t t) {
  const uint64_t* keys = pass_src(rx.dig_hist, 4, n_pad) ? rx.keys_alt : rx.keys;  // after the 4 passes
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
  // the skip decisions are taken on the device (no host round trip mid-step); the host learns
  // the pass count from the histograms afterwards (autx_step_stats), not needed here
  uint32_t passes = 4;
  for (int d = 0; d < 4; ++d) {
    __atomic_fetch_add(&g_kernel_launches, 3ull, __ATOMIC_RELAXED);
    k_hist<<<ntiles, RX_THREADS, 0, s>>>(rx, rx.tile_hist, ntiles, d);
    k_scan_h<<<8, 1024, 0, s>>>(rx, rx.tile_hist, ntiles, d);
    k_scatter<<<ntiles, RX_THREADS, 0, s>>>(rx, rx.tile_hist, ntiles, d);
  }
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_take<<<1, 1024, 0, s>>>(rx, n_pad, ct, ctl, out, pol.max_batch, pol.K, t);
  if (passes_out) *passes_out = passes;
  return cudaGetLastError();
}

}  // namespace autx
