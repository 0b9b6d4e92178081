// Warp/block primitives (scans, segmented scans, bitonic sort) written for sm_100a.
#pragma once
#include <cstdint>
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

template <typename T, int NT>
__device__ __forceinline__ T block_sum(T v, T* smem) {
  T tot;
  block_excl_scan<T, NT>(v, smem, &tot);
  return tot;
}

// ---- segmented inclusive scan (head flags), warp shuffles + one cross-warp pass -------------
struct OpSum {
  template <typename T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
struct OpMax {
  template <typename T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
};

// Inclusive segmented scan over the block in thread order.  `head` marks the first element
// of a segment.  smem_v: >= 32 T, smem_f: >= 32 uint32.
template <typename T, int NT, typename Op>
__device__ __forceinline__ T block_seg_scan(T v, bool head, Op op, T* smem_v, uint32_t* smem_f) {
  uint32_t f = head;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, d);
    uint32_t fu = __shfl_up_sync(0xffffffffu, f, d);
    if (lane_id() >= (uint32_t)d) {
      if (!f) v = op(u, v);
      f |= fu;
    }
  }
  constexpr int NW = NT / 32;
  if (lane_id() == 31) {
    smem_v[warp_id()] = v;
    smem_f[warp_id()] = f;
  }
  __syncthreads();
  if (warp_id() == 0) {
    // exclusive segmented scan of the warp aggregates
    T w = lane_id() < NW ? smem_v[lane_id()] : T(0);
    uint32_t wf = lane_id() < NW ? smem_f[lane_id()] : 1u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      T u = __shfl_up_sync(0xffffffffu, w, d);
      uint32_t fu = __shfl_up_sync(0xffffffffu, wf, d);
      if (lane_id() >= (uint32_t)d) {
        if (!wf) w = op(u, w);
        wf |= fu;
      }
    }
    // shift to exclusive: carry into warp i = inclusive aggregate of warp i-1
    T prev = __shfl_up_sync(0xffffffffu, w, 1);
    uint32_t has = lane_id() > 0;
    if (lane_id() < NW) {
      smem_v[lane_id()] = prev;
      smem_f[lane_id()] = has;
    }
  }
  __syncthreads();
  if (!f && smem_f[warp_id()]) v = op(smem_v[warp_id()], v);
  __syncthreads();
  return v;
}

// ---- bitonic sort of (hi, lo) pairs in shared memory, ascending lexicographic -------------
__device__ __forceinline__ bool pair_gt(uint64_t ah, uint32_t al, uint64_t bh, uint32_t bl) {
  return ah > bh || (ah == bh && al > bl);
}

template <int NT>
__device__ void bitonic_sort_pairs(uint64_t* hi, uint32_t* lo, uint32_t np) {
  for (uint32_t k = 2; k <= np; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < np / 2; i += NT) {
        // index of the lower element of the i-th compare-exchange pair
        uint32_t a = 2 * i - (i & (j - 1));
        uint32_t b = a + j;
        bool up = (a & k) == 0;
        uint64_t ah = hi[a], bh = hi[b];
        uint32_t al = lo[a], bl = lo[b];
        if (pair_gt(ah, al, bh, bl) == up) {
          hi[a] = bh; lo[a] = bl;
          hi[b] = ah; lo[b] = al;
        }
      }
      __syncthreads();
    }
  }
}

// Bitonic sort of exactly 2*NT (key, payload) pairs held two per thread (element i lives in
// thread i/2, slot i%2).  Partner distance j = 1 is a register swap, 2 <= j <= 32 a warp
// shuffle, j >= 64 goes through shared memory (sk/sp: 2*NT entries).  Keys must be unique or
// payload-tied; ascending order on (key, payload).
template <int NT>
__device__ void bitonic_sort_reg2(uint64_t& k0, uint32_t& v0, uint64_t& k1, uint32_t& v1, uint64_t* sk,
                                  uint32_t* sp) {
  constexpr uint32_t N = 2 * NT;
  const uint32_t tid = threadIdx.x;
  for (uint32_t k = 2; k <= N; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j == 1) {
        const bool asc = ((2 * tid) & k) == 0;
        if (pair_gt(k0, v0, k1, v1) == asc) {
          uint64_t tk = k0; k0 = k1; k1 = tk;
          uint32_t tv = v0; v0 = v1; v1 = tv;
        }
      } else if (j <= 32) {
        const uint32_t lanemask = j >> 1;  // partner thread = tid ^ (j/2), same warp
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          uint64_t& kk = r ? k1 : k0;
          uint32_t& vv = r ? v1 : v0;
          const uint32_t i = 2 * tid + r;
          uint64_t pk = __shfl_xor_sync(0xffffffffu, kk, lanemask);
          uint32_t pv = __shfl_xor_sync(0xffffffffu, vv, lanemask);
          const bool asc = (i & k) == 0;
          const bool lower = (i & j) == 0;           // i < partner
          const bool keep_min = lower == asc;
          const bool gt = pair_gt(kk, vv, pk, pv);
          if (keep_min ? gt : !gt) { kk = pk; vv = pv; }
        }
      } else {
        sk[2 * tid] = k0; sp[2 * tid] = v0;
        sk[2 * tid + 1] = k1; sp[2 * tid + 1] = v1;
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          uint64_t& kk = r ? k1 : k0;
          uint32_t& vv = r ? v1 : v0;
          const uint32_t i = 2 * tid + r;
          const uint32_t l = i ^ j;
          uint64_t pk = sk[l];
          uint32_t pv = sp[l];
          const bool asc = (i & k) == 0;
          const bool keep_min = (i < l) == asc;
          const bool gt = pair_gt(kk, vv, pk, pv);
          if (keep_min ? gt : !gt) { kk = pk; vv = pv; }
        }
        __syncthreads();
      }
    }
  }
}

// Block merge sort of 2*NT (key, payload) pairs in shared memory (NT threads, NT a multiple of
// 32, 2*NT a power of two <= 2^16).  Stage 1: every warp sorts its 64 consecutive pairs in
// registers (bitonic, two per lane, shuffles only).  Stage 2: log2(2*NT/64) merge levels; each
// pair finds its output index as (its index in its run) + (its rank in the sibling run), a
// binary search; ties go to the left run, so the merge is stable.  Result in (k, p); (k2, p2)
// is scratch of the same size.  Order: ascending (key, payload).
__device__ __forceinline__ bool kp_less(uint64_t ak, uint32_t ap, uint64_t bk, uint32_t bp) {
  return ak < bk || (ak == bk && ap < bp);
}

template <int NT>
__device__ void block_merge_sort(uint64_t* k, uint32_t* p, uint64_t* k2, uint32_t* p2) {
  constexpr uint32_t N = 2 * NT;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // ---- stage 1: 64-element runs per warp, in registers ----------------------------------
  {
    const uint32_t base = w * 64;
    uint64_t k0 = k[base + 2 * lane], k1 = k[base + 2 * lane + 1];
    uint32_t v0 = p[base + 2 * lane], v1 = p[base + 2 * lane + 1];
    for (uint32_t kk = 2; kk <= 64; kk <<= 1) {
      for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
        if (j == 1) {
          const bool asc = ((2 * lane) & kk) == 0;
          if (kp_less(k1, v1, k0, v0) == asc) {
            uint64_t tk = k0; k0 = k1; k1 = tk;
            uint32_t tv = v0; v0 = v1; v1 = tv;
          }
        } else {
          const uint32_t m = j >> 1;
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            uint64_t& x = r ? k1 : k0;
            uint32_t& y = r ? v1 : v0;
            const uint32_t i = 2 * lane + r;
            uint64_t px = __shfl_xor_sync(0xffffffffu, x, m);
            uint32_t py = __shfl_xor_sync(0xffffffffu, y, m);
            const bool keep_min = ((i & j) == 0) == ((i & kk) == 0);
            const bool take = keep_min ? kp_less(px, py, x, y) : kp_less(x, y, px, py);
            if (take) { x = px; y = py; }
          }
        }
      }
    }
    __syncwarp();
    k[base + 2 * lane] = k0; p[base + 2 * lane] = v0;
    k[base + 2 * lane + 1] = k1; p[base + 2 * lane + 1] = v1;
  }
  __syncthreads();
  // ---- stage 2: merge levels ------------------------------------------------------------
  uint64_t* sk = k; uint32_t* sp = p;
  uint64_t* dk = k2; uint32_t* dp = p2;
  for (uint32_t L = 64; L < N; L <<= 1) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint32_t i = 2 * tid + r;
      const uint32_t run = i / L, off = i % L;
      const uint32_t pair_base = (run & ~1u) * L;
      const bool left = (run & 1u) == 0;
      const uint32_t sib = left ? pair_base + L : pair_base;
      const uint64_t xk = sk[i];
      const uint32_t xp = sp[i];
      // rank in the sibling run: left elements count sibling keys < x (lower bound), right
      // elements count sibling keys <= x (upper bound), which keeps the merge stable
      uint32_t lo = 0, hi = L;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint64_t mk = sk[sib + mid];
        const uint32_t mp = sp[sib + mid];
        const bool before = left ? kp_less(mk, mp, xk, xp) : !kp_less(xk, xp, mk, mp);
        if (before) lo = mid + 1; else hi = mid;
      }
      const uint32_t dst = pair_base + off + lo;
      dk[dst] = xk;
      dp[dst] = xp;
    }
    __syncthreads();
    uint64_t* tk = sk; sk = dk; dk = tk;
    uint32_t* tp = sp; sp = dp; dp = tp;
  }
  if (sk != k) {  // odd number of levels: copy back
    for (uint32_t i = tid; i < N; i += NT) { k[i] = sk[i]; p[i] = sp[i]; }
    __syncthreads();
  }
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

__device__ __forceinline__ uint32_t ceil_div_u32(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

}  // namespace autx
