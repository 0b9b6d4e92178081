// sm_100a kernels of one Autellix scheduling step.  Default chain,
// PDL-linked on one stream:
//
//   k_prologue   (a1, a2)  completion records -> process table (commutative reductions), rows
//                          released; arrivals appended, inherit service, placed in a queue
//   k_scan_bulk  (a4)      dense TMA-staged pass over every call: anti-starvation (integer
//                          cross-multiply) + per-tile / per-super-tile queue counts
//   k_gather_ss  (a5)      q*, m' and each tile's candidate offset from the counts; emits the
//                          candidate set (<= BS rows of the lowest queues, table order) and the
//                          previous batch's records and region-B keys
//   k_rank       (a5)      multi-CTA rank counting of the <= 2 BS unique keys
//   k_finalize   (a5, a6, a3, a7 plan)  prefix cutoff on BS and the KV budget, admit/preempt
//                          lists, step accounting and eager demotion, GPU block allocation and
//                          the swap plan, host mirrors
//
// Every step of Alg. 1 runs here; the host only stages records.  Citations: see autx.h.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "autx_internal.cuh"
#include "block_prims.cuh"
#include "../../include/autx.h"

namespace autx {

__device__ __forceinline__ uint32_t place_queue(const Policy& pol, uint32_t svc) {
  // Alg. 1 l.12, half-open [lo, hi) (R1); FCFS/MLFQ: all new calls enter Q_1.
  if (pol.policy == AUTX_FCFS || pol.policy == AUTX_MLFQ) return 0;
  uint32_t q = 0;
  for (uint32_t i = 0; i + 1 < pol.K; ++i)
    if (svc >= pol.q_hi[i]) q = i + 1;
  return q;
}

#ifdef AUTX_PHASE_SYNC
// profiling build: a barrier that must complete (its result is consumed) before the stamp, so
// deferred-blocking barriers cannot shift time into the next phase
#define STAMP(i) do { if (__syncthreads_count(1) && threadIdx.x == 0) ctl->dbg[i] = globaltimer(); } while (0)
#else
#define STAMP(i) do { if (threadIdx.x == 0) ctl->dbg[i] = globaltimer(); } while (0)
#endif

// Chain stamps (autx_set_timing mode 2, or always in a -DAUTX_CHAIN_STAMPS build): per kernel k
// of the step chain, %globaltimer when CTA 0 passes griddepcontrol.wait (dbg[32 + 3k]), the
// latest CTA end (33 + 3k) and the latest CTA start past the wait (34 + 3k); finalize moves
// dbg[32, 64) to dbg[64, 96) at the step's end.  Off by default: one uniform parameter test.
#ifdef AUTX_CHAIN_STAMPS
#define STAMPS_ON true
#else
#define STAMPS_ON (pol.stamps != 0)
#endif
#define CHAIN_BEGIN(k) do { if (STAMPS_ON && threadIdx.x == 0) { const unsigned long long g_ = globaltimer(); \
    if (blockIdx.x == 0) ctl->dbg[32 + 3 * (k)] = g_; atomicMax(&ctl->dbg[34 + 3 * (k)], g_); } } while (0)
#define CHAIN_END(k) do { if (STAMPS_ON && threadIdx.x == 0) atomicMax(&ctl->dbg[33 + 3 * (k)], globaltimer()); } while (0)

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ceil(tokens / block_tokens) (R14, R28): a shift when block_tokens is a power of two
__device__ __forceinline__ uint32_t blocks_for(const Policy& pol, uint32_t tokens) {
  return pol.bt_shift != 0xFFu ? (tokens + pol.block_tokens - 1) >> pol.bt_shift
                               : (tokens + pol.block_tokens - 1) / pol.block_tokens;
}

// Alg. 1 l.24-26 (R3, R4): W = pwait[p] + wait_c, T = svc[p] + mtime_c; promote iff not 0/0 and
// W * beta_den >= beta_num * T.  Fast path: W and T fit in 32 bits (no carry), so the products
// are single 32x32->64 multiplies; otherwise the 128-bit-exact comparison.
__device__ __forceinline__ bool starving(const Policy& pol, const PInfo& pi, uint32_t wait, uint32_t mtime) {
  const uint32_t W32 = (uint32_t)pi.pwait + wait, T32 = pi.svc + mtime;
  if ((uint32_t)(pi.pwait >> 32) == 0 && W32 >= wait && T32 >= pi.svc)
    return (W32 | T32) != 0 && (uint64_t)W32 * pol.beta_den >= (uint64_t)T32 * pol.beta_num;
  const uint64_t W = pi.pwait + (uint64_t)wait, T = (uint64_t)pi.svc + mtime;
  return !(W == 0 && T == 0) && mul_ge(W, pol.beta_den, T, pol.beta_num);
}

__device__ __forceinline__ void set_err(Ctl* ctl, uint32_t code, uint32_t info) {
  if (atomicCAS(&ctl->err, 0u, code) == 0u) ctl->err_info = info;
}

// ---------------------------------------------------------------------------------------------
// a1: UPDATE_PROCESS_TABLE (Alg. 1 l.1-7) for the calls that finished in step t-1.
//   PLAS (Eq. 1): svc[p] += sum exec;  ATLAS (l.4): svc[p] = max(svc[p], max(inh + exec));
//   pwait[p] += sum totwait (R5), totwait(c) = (t - arr) - exec (active steps not running).
// Each record updates its program's row with one reduction per field (PLAS: add, ATLAS: max;
// pwait: add).  Integer sums and maxima commute, so the row is the same whatever order the records
// arrive in (deterministic), and fire-and-forget reductions put no round trip on the step's path.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void apply_record(const Policy& pol, ProgTable pt, const CompRec& r, uint32_t t) {
  PInfo* pi = pt.info + r.prog;
  if (pol.policy == AUTX_ATLAS || pol.policy == AUTX_ATLAS_EQ2) atomicMax(&pi->svc, r.cp);  // Alg. 1 l.4
  else atomicAdd(&pi->svc, r.exec);                          // Eq. 1
  if (r.tw) atomicAdd(&pi->pwait, (unsigned long long)r.tw);  // Alg. 1 l.5-6, R5
  pt.last_comp[r.prog] = t;
}

template <int NT>
__device__ void complete_body(const Policy& pol, CallTable& ct, ProgTable& pt, Ctl* ctl, const uint32_t* slots,
                              uint32_t n, uint32_t t, KvState& kv, bool kv_on, CompRec* rec_out, bool apply,
                              CompRec* s_rec = nullptr, const uint32_t* lin = nullptr) {
  __shared__ uint32_t red_u[33];
  const uint32_t tid = threadIdx.x;
  STAMP(16);
  for (uint32_t base = 0; base < n; base += NT) {
    uint32_t i = base + tid;
    bool valid = i < n;
    uint32_t s = valid ? slots[i] : 0;
    CompRec r{};
    uint8_t qf0 = QF_DEAD;
    if (valid) {
      uint32_t e = ct.exec[s];
      qf0 = ct.qf[s];  // loaded with the record fields: one round trip
      r.prog = ct.prog[s];
      r.exec = e;
      r.cp = ct.inh[s] + e;
      r.tw = (t - ct.arr[s]) - e;  // totwait: active steps arr..t-1 that did not run
      rec_out[i] = r;
      if (s_rec) s_rec[i] = r;  // the caller's shared-memory copy (n <= NT)
      if (lin) pt.crit[lin[i]] = r.cp;  // AUTX_ATLAS_EQ2: p(c) + t_c, an Eq. 2 operand
    }
    STAMP(17);
    if (apply && valid) apply_record(pol, pt, r, t);
    STAMP(18);
    // release the row and its KV (completed calls ran in step t-1, hence are resident)
    uint32_t nfree = 0, rslot = NONE;
    if (valid) {
      uint8_t qf = qf0;
      if (kv_on && (qf & QF_RES)) {
        rslot = ct.loc[s];
        AUTX_CHECK(rslot < pol.max_batch, "complete: resident slot", rslot);
        nfree = kv.rs_nblk[rslot];
      }
      ct.qf[s] = QF_DEAD;
      ct.loc[s] = NONE;
    }
    if (kv_on) {
      uint32_t tot;
      uint32_t off = block_excl_scan<uint32_t, NT>(nfree, red_u, &tot);
      uint32_t has = rslot != NONE, rtot;
      uint32_t roff = block_excl_scan<uint32_t, NT>(has, red_u, &rtot);
      uint32_t top = ctl->free_top, rtop = ctl->rs_free_top;
      if (rslot != NONE) {
        AUTX_CHECK(nfree == blocks_for(pol, ct.tok[s] + ct.exec[s]), "complete: held blocks", nfree);
        const uint32_t* src = kv.rs_blocks + (size_t)rslot * pol.max_blocks_per_call;
        AUTX_CHECK(top + off + nfree <= pol.n_gpu_blocks, "complete: free stack push", top + off + nfree);
        for (uint32_t j = 0; j < nfree; ++j) kv.free_stack[top + off + j] = src[j];
        kv.rs_nblk[rslot] = 0;
        AUTX_CHECK(rtop + roff < pol.max_batch, "complete: resident-slot push", rtop + roff);
        kv.rs_free[rtop + roff] = rslot;
      }
      __syncthreads();
      if (tid == 0) {
        ctl->free_top = top + tot;
        ctl->rs_free_top = rtop + rtot;
      }
    }
    __syncthreads();
  }
  if (tid == 0) ctl->t = t;
  STAMP(19);
}

template <int NT>
__global__ void __launch_bounds__(NT) k_complete(Policy pol, CallTable ct, ProgTable pt, Ctl* ctl,
                                                 const uint32_t* slots, uint32_t n, uint32_t t, KvState kv,
                                                 bool kv_on, CompRec* rec_out, bool apply) {
  pdl_wait();
  pdl_trigger();
  complete_body<NT>(pol, ct, pt, ctl, slots, n, t, kv, kv_on, rec_out, apply);
}

// Multi-engine: apply every engine's completion records (R22: sums and maxima commute, so the
// replicated tables stay identical whatever the order).  recs of rank r start at
// base + r * stride bytes, after a RouteHdr.
__global__ void __launch_bounds__(FIN_THREADS) k_apply(Policy pol, ProgTable pt, const char* base,
                                                       uint64_t stride, uint32_t G, uint32_t t) {
  for (uint32_t r = 0; r < G; ++r) {
    const RouteHdr* h = reinterpret_cast<const RouteHdr*>(base + r * stride);
    const CompRec* recs = reinterpret_cast<const CompRec*>(h + 1);
    const uint32_t n = h->n_comp;
    for (uint32_t i = threadIdx.x; i < n; i += FIN_THREADS) apply_record(pol, pt, recs[i], t);
  }
}

// The epoch record's header (autx_route): load and completion count from the kernel parameters,
// so the host stages nothing that a later step could overwrite before the copy ran.
__global__ void k_route_hdr(RouteHdr* h, unsigned long long load, uint32_t n_comp) {
  if (threadIdx.x == 0) *h = RouteHdr{load, n_comp, 0u};
}

// Alg. 2 over the replicated arrival batch, canonical order: tokens <= threshold -> argmin load
// (ties -> lowest engine id); else the program's pinned engine, or argmin + pin (l.5-10).  The
// chosen engine's load is incremented after each assignment (R23).  mode 1 (Least Used):
// argmin load for every call, no pins; mode 2 (Round Robin): the replicated cursor *rr.
// One thread: the recurrence through `load` is sequential by definition; G <= 8 loads stay in
// registers.
__global__ void k_route(const char* base, uint64_t stride, uint32_t G, const RouteArr* arr,
                        uint32_t n, int8_t* pin, uint32_t threshold, int32_t* out, uint32_t mode,
                        uint32_t* rr) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (mode == 2) {
    uint32_t e = *rr;
    for (uint32_t i = 0; i < n; ++i) {
      out[i] = (int32_t)e;
      e = e + 1 == G ? 0 : e + 1;
    }
    *rr = e;
    return;
  }
  uint64_t load[8];
#pragma unroll
  for (int e = 0; e < 8; ++e)
    load[e] = e < (int)G ? reinterpret_cast<const RouteHdr*>(base + e * stride)->load : ~0ull;
  for (uint32_t i = 0; i < n; ++i) {
    RouteArr a = arr[i];
    int e;
    const bool lng = mode == 0 && a.tok > threshold;
    int pinned = lng ? pin[a.prog] : -1;
    if (lng && pinned >= 0) {
      e = pinned;
    } else {
      e = 0;
      uint64_t best = load[0];
#pragma unroll
      for (int k = 1; k < 8; ++k)
        if (load[k] < best) { best = load[k]; e = k; }
      if (lng) pin[a.prog] = (int8_t)e;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k == e) load[k] += 1;
    out[i] = e;
  }
}

// ---------------------------------------------------------------------------------------------
// a2: arrivals (Alg. 1 l.9-14).  Rows are appended in canonical order; row index = seq.
// ---------------------------------------------------------------------------------------------
// The call-table row of an arrival that inherits `inh` (Alg. 1 l.11-13); returns its queue.
__device__ __forceinline__ uint32_t register_row(const Policy& pol, CallTable& ct, const ArrivalRec& r, uint32_t s,
                                                 uint32_t t, uint32_t inh) {
  const uint32_t p = r.prog;
  const uint32_t q = place_queue(pol, inh);       // Alg. 1 l.12
  ct.cid[s] = r.cid;
  ct.prog[s] = p;
  ct.arr[s] = t;
  ct.qf[s] = (uint8_t)q;
  ct.base[s] = t;
  ct.mtime[s] = 0;
  ct.exec[s] = 0;
  ct.quanta[s] = pol.quanta[q];                   // Alg. 1 l.13
  ct.inh[s] = inh;
  ct.tok[s] = r.tok;
  ct.loc[s] = NONE;
  ct.hcls[s] = 0;
  return q;
}

__device__ __forceinline__ void register_one(const Policy& pol, CallTable& ct, ProgTable& pt, const ArrivalRec& r,
                                             uint32_t s, uint32_t t, bool have_inh = false, uint32_t inh_given = 0) {
  uint32_t p = r.prog;
  if (r.flags & 2u) {  // first record of a program new in this batch: create its entry
    pt.info[p] = PInfo{0, 0, 0ull};
    pt.last_comp[p] = NONE;
  }
  // Alg. 1 l.11: the service after this step's completions (given by the caller, or read from L2
  // after the caller's fence: see k_prologue)
  uint32_t inh = have_inh ? inh_given : (r.flags & 1u) ? 0u : __ldcg(&pt.info[p].svc);
  pt.last_arr[p] = t;
  register_row(pol, ct, r, s, t, inh);
}

// Eq. 2: p(c_j) = 0 for a root, else max over the parents c_k of p(c_k) + t_k; the
// parents' values were stored at their completion (complete_body), in this kernel before a
// barrier or in an earlier one, hence read from L2.
__device__ __forceinline__ uint32_t eq2_priority(const ProgTable& pt, const uint32_t* par, const ArrivalRec& r) {
  uint32_t p = 0;
  const uint32_t np = r.flags >> 8;
  for (uint32_t k = 0; k < np; ++k) p = max(p, __ldcg(&pt.crit[par[r.par + k]]));
  return p;
}

__global__ void k_register(Policy pol, CallTable ct, ProgTable pt, const ArrivalRec* recs,
                           uint32_t n, uint32_t first_slot, uint32_t t, const uint32_t* par) {
  pdl_wait();
  pdl_trigger();
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const ArrivalRec r = recs[i];
  if (pol.policy == AUTX_ATLAS_EQ2) register_one(pol, ct, pt, r, first_slot + i, t, true, eq2_priority(pt, par, r));
  else register_one(pol, ct, pt, r, first_slot + i, t);
}

// Fused prologue of one step: completions (a1) then arrivals (a2), one CTA; a typical step's
// records travel inside the kernel parameters (no PCIe reads), larger batches through pointers to
// device copies the host made before the step (one DMA each).  256 threads, or 1024 when a batch
// exceeds 256 records (one pass instead of up to four dependent ones).
template <int PRO_THREADS>
__global__ void __launch_bounds__(PRO_THREADS) k_prologue(Policy pol, CallTable ct, ProgTable pt, Ctl* ctl,
                                                          KvState kv, bool kv_on, CompRec* rec_out,
                                                          const PrologueArgs a) {
  __shared__ uint32_t s_comp[PRO_INLINE];
  __shared__ ArrivalRec s_arr[PRO_INLINE];
  const uint32_t tid = threadIdx.x;
  const bool comp_inline = a.n_comp <= PRO_INLINE, arr_inline = a.n_arr <= PRO_INLINE;
  if (comp_inline)
    for (uint32_t i = tid; i < a.n_comp; i += PRO_THREADS) {
      s_comp[i] = a.comp[i];
      // the completions' program rows, which the reductions below read-modify-write: into L2 now,
      // in parallel with the completion rows' loads, instead of one more DRAM round trip after them
      prefetch_l2(&pt.info[a.comp_prog[i]]);
    }
  if (arr_inline)
    for (uint32_t i = tid; i < a.n_arr; i += PRO_THREADS) s_arr[i] = a.arr[i];
  pdl_wait();
  pdl_trigger();
  CHAIN_BEGIN(0);
  if (tid == 0) {  // the step's scalars for the rest of the chain (read after their PDL wait)
    ctl->s_t = a.t;
    ctl->s_n_rows = a.n_rows;
    ctl->s_seqno = a.seqno;
    ctl->s_n_active = a.n_active;
  }
  __syncthreads();
  if (comp_inline && arr_inline) {
    // typical step: arrivals inherit the service after this step's completions (R10) computed
    // here (old row value combined with the step's records of the same program, exactly what the
    // reductions leave in the row), so the row loads go out with the completion loads: one round
    __shared__ CompRec s_rec[PRO_INLINE];
    uint32_t svc_old = 0;
    const bool eq2 = pol.policy == AUTX_ATLAS_EQ2;
    const bool my_arr = tid < a.n_arr;
    if (my_arr && !eq2 && !(s_arr[tid].flags & 1u)) svc_old = __ldcg(&pt.info[s_arr[tid].prog].svc);
    if (a.n_comp)
      complete_body<PRO_THREADS>(pol, ct, pt, ctl, s_comp, a.n_comp, a.t, kv, kv_on, rec_out, true, s_rec,
                                 eq2 ? a.comp_lin : nullptr);
    __syncthreads();
    if (my_arr) {
      const ArrivalRec r = s_arr[tid];
      uint32_t inh = 0;
      if (eq2) {
        inh = eq2_priority(pt, a.par, r);  // parents completed this step are stored above the barrier
      } else if (!(r.flags & 1u)) {
        inh = svc_old;
        for (uint32_t i = 0; i < a.n_comp; ++i)
          if (s_rec[i].prog == r.prog) inh = pol.policy == AUTX_ATLAS ? max(inh, s_rec[i].cp) : inh + s_rec[i].exec;
      }
      register_one(pol, ct, pt, r, a.first_slot + tid, a.t, true, inh);
    }
    CHAIN_END(0);
    return;
  }
  const bool eq2 = pol.policy == AUTX_ATLAS_EQ2;
  if (a.n_comp)
    complete_body<PRO_THREADS>(pol, ct, pt, ctl, comp_inline ? s_comp : a.comp_ptr, a.n_comp, a.t, kv, kv_on,
                               rec_out, true, nullptr, eq2 ? a.comp_lin : nullptr);
  // arrivals inherit the service updated by this step's completions (R10): the reductions are
  // performed at L2 before the barrier releases (fence), and register_one reads svc from L2
  if (a.n_comp && a.n_arr) __threadfence();
  __syncthreads();
  const ArrivalRec* arr = arr_inline ? s_arr : a.arr_ptr;
  for (uint32_t i = tid; i < a.n_arr; i += PRO_THREADS) {
    if (eq2) register_one(pol, ct, pt, arr[i], a.first_slot + i, a.t, true, eq2_priority(pt, a.par, arr[i]));
    else register_one(pol, ct, pt, arr[i], a.first_slot + i, a.t);
  }
  CHAIN_END(0);
}

cudaError_t launch_prologue(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl, KvState kv,
                            bool kv_on, CompRec* rec_out, const PrologueArgs& a) {
  if (std::max(a.n_comp, a.n_arr) > 256)
    return launch_pdl(k_prologue<1024>, 1, 1024, 0, s, pol, ct, pt, ctl, kv, kv_on, rec_out, a);
  return launch_pdl(k_prologue<256>, 1, 256, 0, s, pol, ct, pt, ctl, kv, kv_on, rec_out, a);
}

// ---------------------------------------------------------------------------------------------
// a4 + counting: the dense pass.  Every live call: wait = (t - base) - mtime (every active step
// since the last reset either ran or waited), W = pwait[p] + wait, T = svc[p] + mtime; promote
// to Q_1 iff W * beta_den >= beta_num * T and not 0/0 (Alg. 1 l.24-30, R3/R4/R7).  Demotion
// (l.20-23) was applied eagerly by the previous step's finalize (only batch calls can exhaust a
// quantum, and nothing in between reads q).  Bytes per call: qf 1 + prog 4 + base 4 + mtime 4
// read; a promotion writes base (always: it becomes t) and only the fields that change: qf if
// q != 0, mtime if != 0, quanta if q != 0 or mtime != 0 (a call in Q_1 that has not run since its
// last reset already holds Q_1's quantum).
// ---------------------------------------------------------------------------------------------
// The dense pass runs one tile per CTA, sized for one wave: 256 threads x 8 rows, <= 64
// registers so that 4 CTAs fit per SM (592 tiles = 1.2M rows resident at once).  Every row's
// program-row gather is issued in one round, which is what bounds this latency-bound pass.
// Per-row core of the dense pass over one thread's 8 rows (Alg. 1 l.24-30): program-row gather,
// anti-starvation, promotion writes, queue histogram.
template <int R>
__device__ __forceinline__ void dense_rows(const Policy& pol, CallTable& ct, const ProgTable& pt, uint32_t t,
                                           uint32_t row0, uint32_t (&qfs)[R], const uint32_t (&prog)[R],
                                           uint32_t (&base)[R], uint32_t (&mtim)[R], uint64_t& hq,
                                           uint32_t& npromo, uint32_t& nlive) {
  static_assert(R == 4 || R == 8, "rows per thread");
  const bool anti = pol.beta_den != 0;
  const uint32_t bnum = pol.beta_num, bden = pol.beta_den, quanta0 = pol.quanta[0];
  // the program rows of all 8 rows in one round (svc and pwait only: 12 of the 16 bytes)
  uint32_t svc[R], pwl[R];
  uint32_t big = t & 0x80000000u;  // any operand >= 2^31: this thread needs the exact path
  if (anti) {
    uint32_t pwh[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {  // all gathers first (one round trip), then the corrections
      const bool live = !(qfs[j] & QF_DEAD);
      const uint2 pw = live ? __ldg(reinterpret_cast<const uint2*>(&pt.info[prog[j]].pwait)) : make_uint2(0u, 0u);
      svc[j] = live ? __ldg(&pt.info[prog[j]].svc) : 0u;
      pwl[j] = pw.x;
      pwh[j] = pw.y;
    }
#pragma unroll
    for (int j = 0; j < R; ++j) big |= pwh[j] | ((pwl[j] | svc[j]) & 0x80000000u);
  }
  // Alg. 1 l.24-26 (R3, R4).  With t, svc and pwait below 2^31 (wait, mtime <= t), W and T
  // are below 2^32, so W * beta_den >= beta_num * T is exact as two 32x32->64 products.  A
  // warp holding any larger operand takes the 128-bit comparison (starving()) for all its rows.
  uint32_t stv = 0;  // bit j: row j starving (not 0/0 and the ratio test holds)
  if (anti) {
    // (lanes past n_rows skip this block: vote among the lanes present; each lane still sees
    // its own operand, so the choice is exact whichever lanes take part)
    if (__any_sync(__activemask(), big != 0)) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const bool live = !(qfs[j] & QF_DEAD);
        const PInfo pi = live ? pt.info[prog[j]] : PInfo{0, 0, 0ull};
        stv |= starving(pol, pi, t - base[j] - mtim[j], mtim[j]) ? 1u << j : 0u;
      }
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const uint32_t W = pwl[j] + (t - base[j] - mtim[j]), T = svc[j] + mtim[j];
        const bool st = (W | T) != 0 && (uint64_t)W * bden >= (uint64_t)T * bnum;
        stv |= st ? 1u << j : 0u;
      }
    }
  }
  bool wq = false, wb = false, wm = false;
  if (pol.multistep) {
    // R32: demotions deferred from window steps (quantum exhausted, QF_DEM) happen here, at the
    // scheduling point, before anti-starvation (Alg. 1 l.20-23 before l.24-30, R9); the ratio
    // above does not read q
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const uint32_t qf = qfs[j];
      if ((qf & (QF_DEM | QF_DEAD)) == QF_DEM) {
        const uint32_t q = min((qf & QF_QMASK) + 1u, pol.K - 1);
        ct.quanta[row0 + j] = pol.quanta[q];
        qfs[j] = (qf & ~(uint32_t)(QF_QMASK | QF_DEM)) | q;
        wq = true;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const uint32_t qf = qfs[j];
    const bool live = !(qf & QF_DEAD);
    uint32_t q = qf & QF_QMASK;
    const bool pr = live && ((stv >> j) & 1u);  // Alg. 1 l.26
    if (pr && (q | mtim[j])) ct.quanta[row0 + j] = quanta0;
    wq |= pr && q != 0;
    wm |= pr && mtim[j] != 0;
    wb |= pr;
    qfs[j] = pr ? (qf & ~(uint32_t)QF_QMASK) : qf;
    mtim[j] = pr ? 0u : mtim[j];
    base[j] = pr ? t : base[j];
    q = pr ? 0u : q;
    npromo += pr ? 1u : 0u;
    nlive += live ? 1u : 0u;
    hq += live ? (1ull << (4 * q)) : 0ull;
  }
  if (wq) {
#pragma unroll
    for (int h = 0; h < R / 4; ++h)
      reinterpret_cast<uint32_t*>(ct.qf + row0)[h] =
          qfs[4 * h] | (qfs[4 * h + 1] << 8) | (qfs[4 * h + 2] << 16) | (qfs[4 * h + 3] << 24);
  }
  if (wb) {
#pragma unroll
    for (int h = 0; h < R / 4; ++h)
      reinterpret_cast<uint4*>(ct.base + row0)[h] = make_uint4(base[4 * h], base[4 * h + 1], base[4 * h + 2], base[4 * h + 3]);
  }
  if (wm) {
#pragma unroll
    for (int h = 0; h < R / 4; ++h)
      reinterpret_cast<uint4*>(ct.mtime + row0)[h] = make_uint4(mtim[4 * h], mtim[4 * h + 1], mtim[4 * h + 2], mtim[4 * h + 3]);
  }
}

// Per-tile and per-super-tile queue counts + promotion / live totals of one CTA.
template <int NT = SCAN_THREADS>
__device__ __forceinline__ void tile_counts(const Policy& pol, Ctl* ctl, Outputs& out, uint32_t tile, uint64_t hq,
                                            uint32_t npromo, uint32_t nlive, uint32_t* s_cnt_out = nullptr) {
  constexpr int NW = NT / 32;
  __shared__ uint32_t wq16[NW][MAX_K / 2];  // per warp: 16-bit counts of queues 2w, 2w + 1
  __shared__ uint32_t wn[NW];
  const uint32_t tid = threadIdx.x;
  // per-queue counts: the 4-bit per-thread fields widened to 16 bits (<= 256 per warp), two
  // queues per word, one redux.sync per word of the K queues in use
  const uint32_t K = pol.K;
#pragma unroll
  for (int w = 0; w < MAX_K / 2; ++w) {
    if ((uint32_t)(2 * w) < K) {
      const uint32_t f = (uint32_t)(hq >> (8 * w));
      const uint32_t v = __reduce_add_sync(0xffffffffu, (f & 0xFu) | ((f & 0xF0u) << 12));
      if (lane_id() == 0) wq16[warp_id()][w] = v;
    }
  }
  const uint32_t pl = __reduce_add_sync(0xffffffffu, (npromo << 16) | nlive);  // <= 256 each per warp
  if (lane_id() == 0) wn[warp_id()] = pl;
  __syncthreads();
  if (tid < MAX_K) {
    uint32_t c = 0;
    if (tid < K) {
#pragma unroll
      for (int w = 0; w < NW; ++w) c += (wq16[w][tid >> 1] >> (16 * (tid & 1))) & 0xFFFFu;
    }
    out.tile_cnt[(size_t)tile * MAX_K + tid] = c;
    if (s_cnt_out) s_cnt_out[tid] = c;
    else if (c) atomicAdd(out.sup_cnt + (tile / SUP_TILES) * MAX_K + tid, c);
  } else if (tid == 32) {
    uint32_t a = 0, b = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) { a += wn[w] >> 16; b += wn[w] & 0xFFFFu; }
    uint32_t* qp = ctl->qpart[blockIdx.x % QP_LINES];
    if (a) atomicAdd(qp + MAX_K, a);
    if (b) atomicAdd(qp + MAX_K + 1, b);
  }
}

// pre (A/B switch AUTX_SCAN_PRE): what a CTA does while it waits for the prologue (PDL).  Rows
// below first_new (this step's first arrival slot) keep prog/base/mtime through the prologue
// (it writes only new rows and the qf/loc of completed ones; everything earlier in the stream
// is complete once this grid runs), so they may be read before the wait; qf, the program rows
// and new rows are read after it.  0: nothing early; 1: prog early + L2 prefetch of the rows'
// program entries and of the previous batch's records (the gather's cold reads); 2: prog, base
// and mtime early + the same prefetches.
__global__ void __launch_bounds__(SCAN_THREADS, 4) k_scan_tile(Policy pol, CallTable ct, ProgTable pt, Ctl* ctl,
                                                               Outputs out, uint32_t pre) {
  const uint32_t tid = threadIdx.x, tile = blockIdx.x;
  const uint32_t row0 = tile * TILE + tid * ROWS_PER_THREAD;
  const uint32_t first_new = ctl->s_tail_prev;  // written before this step's chain
  const bool early = pre != 0 && row0 + ROWS_PER_THREAD <= first_new;
  uint4 p0, p1, b0, b1, m0, m1;
  if (early) {
    p0 = __ldcs(reinterpret_cast<const uint4*>(ct.prog + row0));
    p1 = __ldcs(reinterpret_cast<const uint4*>(ct.prog + row0 + 4));
    if (pre >= 2) {
      b0 = __ldcs(reinterpret_cast<const uint4*>(ct.base + row0));
      b1 = __ldcs(reinterpret_cast<const uint4*>(ct.base + row0 + 4));
      m0 = __ldcs(reinterpret_cast<const uint4*>(ct.mtime + row0));
      m1 = __ldcs(reinterpret_cast<const uint4*>(ct.mtime + row0 + 4));
    }
  }
  if (pre != 0) {
    // the previous batch's records: region B and most of region A in the gather
    const uint32_t i = (gridDim.x - 1 - tile) * SCAN_THREADS + tid;
    if (i < ctl->n_prev) {
      const uint32_t sl = out.prev_slots[i];
      prefetch_l2(ct.cid + sl); prefetch_l2(ct.arr + sl); prefetch_l2(ct.tok + sl);
      prefetch_l2(ct.exec + sl); prefetch_l2(ct.mtime + sl); prefetch_l2(ct.quanta + sl);
      prefetch_l2(ct.bidx + sl); prefetch_l2(ct.qf + sl);
    }
    if (early && pol.beta_den != 0) {
      const uint32_t pr[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j == 0 || pr[j] != pr[j - 1]) prefetch_l2(pt.info + pr[j]);
    }
  }
  pdl_wait();
  pdl_trigger();
  CHAIN_BEGIN(1);
  const uint32_t t = ctl->s_t, n_rows = ctl->s_n_rows;
  uint64_t hq = 0;
  uint32_t npromo = 0, nlive = 0;
  if (row0 < n_rows) {
    const uint2 qv = __ldcs(reinterpret_cast<const uint2*>(ct.qf + row0));
    if (!early) {
      p0 = __ldcs(reinterpret_cast<const uint4*>(ct.prog + row0));
      p1 = __ldcs(reinterpret_cast<const uint4*>(ct.prog + row0 + 4));
    }
    if (!early || pre < 2) {
      b0 = __ldcs(reinterpret_cast<const uint4*>(ct.base + row0));
      b1 = __ldcs(reinterpret_cast<const uint4*>(ct.base + row0 + 4));
      m0 = __ldcs(reinterpret_cast<const uint4*>(ct.mtime + row0));
      m1 = __ldcs(reinterpret_cast<const uint4*>(ct.mtime + row0 + 4));
    }
    uint32_t qfs[8], prog[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
    uint32_t base[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    uint32_t mtim[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) qfs[j] = ((j < 4 ? qv.x : qv.y) >> (8 * (j & 3))) & 0xffu;
    dense_rows<8>(pol, ct, pt, t, row0, qfs, prog, base, mtim, hq, npromo, nlive);
  }
  tile_counts(pol, ctl, out, tile, hq, npromo, nlive);
  CHAIN_END(1);
}

// ---------------------------------------------------------------------------------------------
// Dense pass that also emits region A's raw material (AUTX_PIPELINE=sel; the default keeps
// k_gather_ss + k_rank): every tile learns, per queue, how many live calls of that queue the
// earlier tiles hold, saturated at the resident capacity BS (single-pass decoupled look-back,
// tiles taken by ticket so that every tile waited on has started), and writes each live call
// whose rank inside its queue is below BS to cq[q][rank].  Region A is then the concatenation of
// cq[q] for q < q* and the first m' of cq[q*]; the finalize reads q*, m' from the last tile's
// inclusive prefix.  Only the first BS calls of each queue are ever emitted, so the pass writes
// O(K BS) records whatever the table size.
//   Look-back word (one per 4 queues and tile): four 13-bit saturated counts (bits 0, 13, 26, 39;
//   BS <= 2048, so a sum of two fits before it is clamped) and a 2-bit flag (62-63): 0 = not yet,
//   1 = this tile's own counts, 2 = inclusive prefix.  The word carries its own data, so a relaxed
//   load needs no fence.  The finalize zeroes the words after the step.
// ---------------------------------------------------------------------------------------------
constexpr unsigned long long LB_AGG = 1ull << 62, LB_PRE = 2ull << 62, LB_VAL = (1ull << 52) - 1;
constexpr uint32_t LB_SPIN_LIMIT = 1u << 22;
__device__ __forceinline__ unsigned long long lb_sat(unsigned long long v, uint32_t cap) {
  unsigned long long r = 0;
#pragma unroll
  for (int f = 0; f < 4; ++f) r |= (unsigned long long)min((uint32_t)(v >> (13 * f)) & 0x1FFFu, cap) << (13 * f);
  return r;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(SCAN_THREADS, 4) k_scan_emit(Policy pol, CallTable ct, ProgTable pt, Ctl* ctl,
                                                               Outputs out, uint32_t pre) {
  constexpr uint32_t FULL = 0xffffffffu;
  __shared__ uint32_t s_tile, s_emit, s_ne;
  __shared__ uint32_t s_es[TILE], s_er[TILE];  // emitted rows: slot; queue << 16 | rank
  __shared__ uint32_t s_cnt[MAX_K];
  __shared__ unsigned long long s_ex[4];  // this tile's exclusive prefix words
  __shared__ unsigned long long red64[33];
  const uint32_t tid = threadIdx.x, lane = lane_id(), w = warp_id();
  if (tid == 0) { s_tile = atomicAdd(&ctl->scan_ticket, 1u); s_ne = 0; }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t row0 = tile * TILE + tid * ROWS_PER_THREAD;
  const uint32_t first_new = ctl->s_tail_prev;  // written before this step's chain
  const bool early = pre != 0 && row0 + ROWS_PER_THREAD <= first_new;
  uint4 p0, p1;
  if (early) {
    p0 = __ldcs(reinterpret_cast<const uint4*>(ct.prog + row0));
    p1 = __ldcs(reinterpret_cast<const uint4*>(ct.prog + row0 + 4));
    if (pol.beta_den != 0) {
      const uint32_t pr[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j == 0 || pr[j] != pr[j - 1]) prefetch_l2(pt.info + pr[j]);
    }
  }
  pdl_wait();
  pdl_trigger();
  CHAIN_BEGIN(1);
  const uint32_t t = ctl->s_t, n_rows = ctl->s_n_rows;
  const uint32_t K = pol.K, cap = pol.max_batch, nwd = (K + 3) / 4;
  uint64_t hq = 0;
  uint32_t npromo = 0, nlive = 0;
  uint32_t qfs[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) qfs[j] = QF_DEAD;
  if (row0 < n_rows) {
    const uint2 qv = __ldcs(reinterpret_cast<const uint2*>(ct.qf + row0));
    if (!early) {
      p0 = __ldcs(reinterpret_cast<const uint4*>(ct.prog + row0));
      p1 = __ldcs(reinterpret_cast<const uint4*>(ct.prog + row0 + 4));
    }
    const uint4 b0 = __ldcs(reinterpret_cast<const uint4*>(ct.base + row0));
    const uint4 b1 = __ldcs(reinterpret_cast<const uint4*>(ct.base + row0 + 4));
    const uint4 m0 = __ldcs(reinterpret_cast<const uint4*>(ct.mtime + row0));
    const uint4 m1 = __ldcs(reinterpret_cast<const uint4*>(ct.mtime + row0 + 4));
    uint32_t prog[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
    uint32_t base[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    uint32_t mtim[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) qfs[j] = ((j < 4 ? qv.x : qv.y) >> (8 * (j & 3))) & 0xffu;
    dense_rows<8>(pol, ct, pt, t, row0, qfs, prog, base, mtim, hq, npromo, nlive);
  }
  tile_counts(pol, ctl, out, tile, hq, npromo, nlive, s_cnt);
  __syncthreads();
  // publish this tile's counts (tile 0: they are its inclusive prefix), then look back
  // (lane 0 of warp w owns word w: its own-count store precedes its prefix store)
  if (w < nwd && lane == 0) {
    unsigned long long own = 0;
#pragma unroll
    for (int f = 0; f < 4; ++f) own |= (unsigned long long)min(s_cnt[4 * w + f], cap) << (13 * f);
    st_relaxed_u64(out.lb + (size_t)tile * 4 + w, own | (tile == 0 ? LB_PRE : LB_AGG));
    if (tile == 0) s_ex[w] = 0;
  }
  if (tile > 0 && w < nwd) {
    // warp w looks back over word w, 32 predecessors per round, to the nearest inclusive prefix
    // (measured: a block-wide 256-tile window was slower, 17 vs 11.7 us for the pass)
    unsigned long long acc = 0;
    int32_t base = (int32_t)tile;
    uint32_t spins = 0;
    while (true) {
      const int32_t p = base - 1 - (int32_t)lane;
      unsigned long long v = p >= 0 ? ld_relaxed_u64(out.lb + (size_t)p * 4 + w) : LB_PRE;
      while (!__all_sync(FULL, (v >> 62) != 0)) {
        if ((v >> 62) == 0) v = ld_relaxed_u64(out.lb + (size_t)p * 4 + w);
        if (++spins > LB_SPIN_LIMIT && (v >> 62) == 0) {  // a predecessor never published: fail the step
          set_err(ctl, AUTX_E_CUDA, 0xB0000000u | tile);
          v = LB_PRE;
        }
      }
      const uint32_t pm = __ballot_sync(FULL, (v >> 62) == 2);
      const uint32_t upto = pm ? __ffs(pm) - 1 : 31;
      unsigned long long x = lane <= upto ? (v & LB_VAL) : 0ull;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) x = lb_sat(x + __shfl_xor_sync(FULL, x, d), cap);
      acc = lb_sat(acc + x, cap);
      if (pm) break;
      base -= 32;
    }
    if (lane == 0) {
      unsigned long long o = 0;
#pragma unroll
      for (int f = 0; f < 4; ++f) o |= (unsigned long long)min(s_cnt[4 * w + f], cap) << (13 * f);
      s_ex[w] = acc;
      st_relaxed_u64(out.lb + (size_t)tile * 4 + w, lb_sat(acc + o, cap) | LB_PRE);
    }
  }
  __syncthreads();
  // queues this tile emits: live calls here and fewer than BS before it
  if (tid < 32) {
    const uint32_t ex = tid < K ? (uint32_t)(s_ex[tid >> 2] >> (13 * (tid & 3))) & 0x1FFFu : cap;
    const uint32_t b = __ballot_sync(FULL, tid < K && s_cnt[tid] > 0 && ex < cap);
    if (tid == 0) s_emit = b;
  }
  __syncthreads();
  const uint32_t emit = s_emit;
  if (emit) {
    // rank of each of this thread's rows inside its queue: the earlier tiles (s_ex), the earlier
    // threads (block scans of 16-bit fields, 4 queues per scan), the earlier rows of this thread
    for (uint32_t g = 0; g < nwd; ++g) {
      if (!((emit >> (4 * g)) & 0xFu)) continue;
      unsigned long long v = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t q = qfs[j] & QF_QMASK;
        if (!(qfs[j] & QF_DEAD) && (q >> 2) == g) v += 1ull << (16 * (q & 3));
      }
      unsigned long long ex = block_excl_scan<unsigned long long, SCAN_THREADS>(v, red64, nullptr);
      const unsigned long long exw = s_ex[g];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t q = qfs[j] & QF_QMASK;
        if (!(qfs[j] & QF_DEAD) && (q >> 2) == g) {
          const uint32_t f = q & 3;
          const uint32_t r = ((uint32_t)(exw >> (13 * f)) & 0x1FFFu) + ((uint32_t)(ex >> (16 * f)) & 0xFFFFu);
          ex += 1ull << (16 * f);
          if (((emit >> q) & 1u) && r < cap) {
            // the emitted rows go through a shared-memory list so that one thread loads one
            // record (all in one round, no per-row register arrays in this 64-register kernel)
            const uint32_t pos = atomicAdd(&s_ne, 1u);
            s_es[pos] = row0 + j;
            s_er[pos] = q << 16 | r;
          }
        }
      }
    }
    __syncthreads();
    const uint32_t ne = s_ne;
    for (uint32_t i = tid; i < ne; i += SCAN_THREADS) {
      const uint32_t sl = s_es[i], qr = s_er[i];
      CandRec r;
      r.cid = ct.cid[sl];
      r.slot = sl;
      r.arr = ct.arr[sl];
      r.tok = ct.tok[sl];
      r.exec = ct.exec[sl];
      r.mtime = ct.mtime[sl];    // the dense pass's writes (this CTA, before the barriers above)
      r.quanta = ct.quanta[sl];
      r.qf = ct.qf[sl];
      r._pad = (r.qf & QF_RES) ? ct.bidx[sl] : NONE;  // previous resident index
      out.cq[(size_t)(qr >> 16) * cap + (qr & 0xFFFFu)] = r;
    }
  }
  CHAIN_END(1);
}

// Self-selecting gather (default): no separate selection kernel.  Every CTA derives q* and m'
// from the per-queue totals, and a tile CTA its candidate offset from the counts of the earlier
// tiles, both from a two-level table the scan fills: per-tile counts (tile_cnt) and per-super-tile
// counts (sup_cnt, SUP_TILES tiles each, accumulated with atomics).  The prefix of tile T is the
// super-tiles before T's plus the <= SUP_TILES - 1 tiles of T's super-tile before T: one round of
// a few loads per thread (half-warp h, lane k = queue k).
//     off(T) = pre_a(T) + min(pre_q(T), m'),   pre_a = sum_{T'<T} sum_{k<q*} cnt,  pre_q = sum_{T'<T} cnt_q*.
// Inside the tile, a thread's first candidate position follows from the exclusive counts of
// earlier threads (A = live rows with q < q*, Q = live rows of q*) without a second scan, since
// the q* rows are taken in table order:  pos = off + A + min(Q, m' - min(pre_q, m')).
// The thread taking the m'-th q* row publishes its slot (region A's boundary); the previous-batch
// CTAs emit keys for every live q* call of the previous batch and k_rank drops those with
// slot <= boundary (they are in region A).
__device__ __forceinline__ void gather_ss_body(Policy& pol, CallTable& ct, Ctl* ctl, Outputs& out, uint32_t n_rows, uint32_t ntiles, uint32_t t) {
  constexpr int NT = SCAN_THREADS, NW = NT / 32, NH = NT / MAX_K;  // NH half-warps of MAX_K lanes
  __shared__ uint32_t s_tot[NH][MAX_K], s_pre[NH][MAX_K];
  __shared__ uint32_t s_qs, s_m, s_prea, s_preq, s_has;
  __shared__ uint32_t s_own[MAX_K];
  __shared__ uint32_t s_cnt[NW];
  const uint32_t tid = threadIdx.x, tile = blockIdx.x;
  const uint32_t K = pol.K, BS = pol.max_batch;
  const bool is_tile = tile < ntiles;
  // (1) one round of independent loads: this tile's queue bytes first (they do not depend on the
  // selection), then the counts
  const uint32_t row0 = tile * TILE + tid * ROWS_PER_THREAD;
  const uint2 qv = is_tile && row0 < n_rows ? *reinterpret_cast<const uint2*>(ct.qf + row0)
                                            : make_uint2(0x40404040u, 0x40404040u);
  {
    const uint32_t h = tid / MAX_K, k = tid % MAX_K;
    const uint32_t nsup = (ntiles + SUP_TILES - 1) / SUP_TILES, my_sup = tile / SUP_TILES;
    uint32_t tot = 0, pre = 0;
    if (k < K) {
      // all loads issued before any is consumed (a rolled loop would chain one L2 round trip per
      // iteration): the tile count, then up to 8 super-tile rows per half-warp (4.2M rows)
      const uint32_t tr = my_sup * SUP_TILES + h;  // earlier tile of the same super-tile, or this one
      const bool has_tr = is_tile && tr <= tile;
      const uint32_t c = has_tr ? __ldcg(out.tile_cnt + (size_t)tr * MAX_K + k) : 0u;
      constexpr int SU = 8;
      uint32_t v[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const uint32_t S = h + u * NH;
        v[u] = S < nsup ? __ldcg(out.sup_cnt + S * MAX_K + k) : 0u;
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const uint32_t S = h + u * NH;
        tot += v[u];
        pre += (is_tile && S < my_sup) ? v[u] : 0u;
      }
      for (uint32_t S = h + SU * NH; S < nsup; S += NH) {  // larger tables
        const uint32_t w = __ldcg(out.sup_cnt + S * MAX_K + k);
        tot += w;
        pre += (is_tile && S < my_sup) ? w : 0u;
      }
      if (has_tr) {
        if (tr < tile) pre += c;
        else s_own[k] = c;
      }
    }
    s_tot[h][k] = tot;
    s_pre[h][k] = pre;
    if (tile == 0 && tid < 32) {
      // promotions (even lanes) and live rows (odd lanes) for finalize's host record
      uint32_t stat = tid < 2 * QP_LINES ? __ldcg(&ctl->qpart[tid >> 1][MAX_K + (tid & 1)]) : 0u;
#pragma unroll
      for (int d = 2; d < 32; d <<= 1) stat += __shfl_xor_sync(0xffffffffu, stat, d);
      if (tid == 0) ctl->n_promoted = stat;
      if (tid == 1) ctl->n_live = stat;
    }
  }
  if (!is_tile) {
    // previous batch: records (for preempt) and region-B keys
    const uint32_t j = (tile - ntiles) * NT + tid;
    const uint32_t n_prev = ctl->n_prev;
    CandRec r;
    if (j < n_prev) load_rec(ct, out.prev_slots[j], &r);
    __syncthreads();
    if (tid < 32) {
      uint32_t tq = 0;
      if (tid < MAX_K) {
#pragma unroll
        for (int h = 0; h < NH; ++h) tq += s_tot[h][tid];
      }
      const uint32_t incl = warp_incl_scan(tq);
      const uint32_t b = __ballot_sync(0xffffffffu, tid < K && incl >= BS);
      const uint32_t qs = b ? __ffs(b) - 1 : K;
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      if (tid == 0) { s_qs = qs; s_m = qs < K ? BS : tot; }  // s_m: n_cand_a here
    }
    __syncthreads();
    if (j < n_prev) {
      out.prev_rec[j] = r;
      const bool b = !(r.qf & QF_DEAD) && (r.qf & QF_QMASK) == s_qs;
      out.ckey[s_m + j] = b ? cand_key(r, t) : ~0ull;
      out.ckvb[s_m + j] = blocks_for(pol, r.tok + r.exec + 1);  // R14
    }
    return;
  }
  __syncthreads();
  // (2) q*, m', and this tile's prefix (warp 0, lane k = queue k)
  if (tid < 32) {
    uint32_t tq = 0, pk = 0;
    if (tid < MAX_K) {
#pragma unroll
      for (int h = 0; h < NH; ++h) { tq += s_tot[h][tid]; pk += s_pre[h][tid]; }
    }
    const uint32_t incl = warp_incl_scan(tq);
    const uint32_t b = __ballot_sync(0xffffffffu, tid < K && incl >= BS);
    const uint32_t qs = b ? __ffs(b) - 1 : K;
    const uint32_t excl = __shfl_sync(0xffffffffu, incl - tq, qs & 31);
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t pa = warp_sum(tid < qs ? pk : 0u);
    const uint32_t pq = __shfl_sync(0xffffffffu, pk, qs & 31);
    // this tile's own live rows below q* and of q*: no candidate unless one of them is taken
    const uint32_t own = tid < K ? s_own[tid] : 0u;
    const uint32_t oa = warp_sum(tid < qs ? own : 0u);
    const uint32_t oq = __shfl_sync(0xffffffffu, own, qs & 31);
    if (tid == 0) {
      const uint32_t m = qs < K ? BS - excl : 0;
      s_qs = qs;
      s_m = m;
      s_prea = pa;
      s_preq = qs < K ? pq : 0;
      s_has = oa > 0 || (qs < K && oq > 0 && pq < m);
      if (tile == 0) {
        ctl->qstar = qs;
        ctl->mprime = m;
        ctl->n_cand_a = qs < K ? BS : tot;
      }
    }
  }
  __syncthreads();
  // tiles without candidates leave now (their SM slots go to the next kernel's CTAs); the
  // boundary row is always in a tile with candidates
  if (STAMPS_ON && tile == 0 && tid == 0) ctl->dbg[57] = globaltimer();
  if (tid == 0 && out.gtile) out.gtile[tile] = s_has;
  if (!s_has) return;
  const uint32_t qs = s_qs, m = s_m;
  uint32_t qfs[8], na = 0, nq = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    qfs[j] = ((j < 4 ? qv.x : qv.y) >> (8 * (j & 3))) & 0xffu;
    const bool live = !(qfs[j] & QF_DEAD);
    const uint32_t q = qfs[j] & QF_QMASK;
    na += (live && q < qs) ? 1u : 0u;
    nq += (live && q == qs) ? 1u : 0u;
  }
  // (3) exclusive (A, Q) counts of the earlier threads of this tile
  const uint32_t v = (na << 16) | nq;  // <= 2048 each
  const uint32_t vin = warp_incl_scan(v);
  if (lane_id() == 31) s_cnt[warp_id()] = vin;
  __syncthreads();
  uint32_t vex = vin - v;
#pragma unroll
  for (int w = 0; w < NW; ++w) vex += (uint32_t)w < warp_id() ? s_cnt[w] : 0u;
  const uint32_t pre_a = s_prea, pre_q = s_preq;
  const uint32_t mq = m - min(pre_q, m);  // q* rows still to take at this tile's start
  uint32_t rq = pre_q + (vex & 0xffffu);
  uint32_t pos = pre_a + min(pre_q, m) + (vex >> 16) + min(vex & 0xffffu, mq);
  uint32_t flags = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t qf = qfs[j];
    if (qf & QF_DEAD) continue;
    const uint32_t q = qf & QF_QMASK;
    bool sel = q < qs;
    if (q == qs) {
      sel = rq < m;
      if (rq + 1 == m) ctl->qs_bnd1 = row0 + j + 1;
      ++rq;
    }
    if (sel) flags |= 1u << j;
  }
  if (STAMPS_ON && tile == 0 && tid == 0) ctl->dbg[58] = globaltimer();
  if (flags) {
    const uint4* cidv = reinterpret_cast<const uint4*>(ct.cid + row0);
    uint4 c4[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) c4[w] = cidv[w];
    uint4 ar[2], tk[2], ex[2], mt[2], qt[2], bd[2];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      ar[w] = reinterpret_cast<const uint4*>(ct.arr + row0)[w];
      tk[w] = reinterpret_cast<const uint4*>(ct.tok + row0)[w];
      ex[w] = reinterpret_cast<const uint4*>(ct.exec + row0)[w];
      mt[w] = reinterpret_cast<const uint4*>(ct.mtime + row0)[w];
      qt[w] = reinterpret_cast<const uint4*>(ct.quanta + row0)[w];
      bd[w] = reinterpret_cast<const uint4*>(ct.bidx + row0)[w];
    }
    auto lane4 = [](const uint4& a, int k) { return k == 0 ? a.x : k == 1 ? a.y : k == 2 ? a.z : a.w; };
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (flags & (1u << j)) {
        CandRec r;
        const uint4& cc = c4[j >> 1];
        r.cid = (j & 1) ? ((uint64_t)cc.w << 32 | cc.z) : ((uint64_t)cc.y << 32 | cc.x);
        r.slot = row0 + j;
        r.arr = lane4(ar[j >> 2], j & 3);
        r.tok = lane4(tk[j >> 2], j & 3);
        r.exec = lane4(ex[j >> 2], j & 3);
        r.mtime = lane4(mt[j >> 2], j & 3);
        r.quanta = lane4(qt[j >> 2], j & 3);
        r.qf = qfs[j];
        r._pad = (qfs[j] & QF_RES) ? lane4(bd[j >> 2], j & 3) : NONE;  // previous resident index
        out.cand[pos] = row0 + j;
        out.cand_rec[pos] = r;
        out.ckey[pos] = cand_key(r, t);
        out.ckvb[pos] = blocks_for(pol, r.tok + r.exec + 1);  // R14
        ++pos;
      }
  }
  if (STAMPS_ON && tile == 0) {
    __syncwarp();
    if (tid == 0) ctl->dbg[59] = globaltimer();
  }
}

__global__ void __launch_bounds__(SCAN_THREADS, 4) k_gather_ss(Policy pol, CallTable ct, Ctl* ctl, Outputs out) {
  // a tile that held candidates in the previous step likely holds them again (region A is the
  // head of q* in table order): pull its record columns into L2 while the dense pass runs, so
  // that the emission below reads them from L2 instead of DRAM (2 prefetches per thread)
  if (out.gtile && blockIdx.x < out.gtile_cap && out.gtile[blockIdx.x]) {
    const size_t r0 = (size_t)blockIdx.x * TILE;
#pragma unroll
    for (uint32_t k = 0; k < 2; ++k) {  // 128-B lines: 128 of cid, then 64 of each 4-byte column
      const uint32_t L = threadIdx.x + k * SCAN_THREADS;
      if (L < 128) {
        prefetch_l2(ct.cid + r0 + 16 * L);
      } else {
        const uint32_t c = (L - 128) >> 6, o = 32 * ((L - 128) & 63);
        const uint32_t* col = c == 0 ? ct.arr : c == 1 ? ct.tok : c == 2 ? ct.exec : c == 3 ? ct.mtime : c == 4 ? ct.quanta : ct.bidx;
        prefetch_l2(col + r0 + o);
      }
    }
  }
  pdl_wait();
  pdl_trigger();
  const uint32_t t = ctl->s_t, n_rows = ctl->s_n_rows;
  const uint32_t ntiles = n_rows ? (n_rows + TILE - 1) / TILE : 1u;
  CHAIN_BEGIN(3);
  gather_ss_body(pol, ct, ctl, out, n_rows, ntiles, t);
  CHAIN_END(3);
}

// ---------------------------------------------------------------------------------------------
// a5/a6/a3/a7-plan: one CTA.  Sort <= 2 BS candidate keys
//     q:4 | arrival (relative to t):27 | not-running:1 | seq (row):31       (R11, R12)
// (region A from the gather, plus the previous batch's calls of q*, de-duplicated), cut the
// longest prefix with count <= BS and sum kvb <= P (Alg. 1 l.32-39, first misfit stops, R13),
// emit batch/admit/preempt, account (batch: exec++, mtime++, quanta--, running; everyone else
// waits implicitly via the closed-form counters), demote batch calls whose quantum is exhausted
// (Alg. 1 l.20-23), allocate KV blocks and build the swap plan.
// ---------------------------------------------------------------------------------------------
extern __shared__ unsigned char fin_smem[];
template <int NT, int R, bool LISTS = false, bool ORD = false, bool SEL = false>
__device__ void finalize_body(const Policy& pol, CallTable& ct, Ctl* ctl, Outputs& out, KvState& kv, bool kv_on,
                              uint32_t t, uint32_t np, uint32_t seqno, const CandRec (&pp)[R], uint32_t n_prev_pre);

__device__ __forceinline__ uint32_t ceil_log2(uint32_t x) { return x <= 1 ? 0 : 32 - __clz(x - 1); }

// k_rank: the candidates' sort.  A single SM needs ~35k cycles to sort 2048 64-bit keys with
// any block sort (measured: scripts/micro/sort_bench.cu), so the order is computed across many
// SMs instead: every CTA holds all n <= 2 BS keys in shared memory and each key's output index is
// the number of keys before it (the keys are unique), RANK_SUB threads per key.
// 16 keys per CTA; AUTX_RANK_THREADS threads per CTA (RANK_SUB per key, twice that per key in the
// wide mode): more warps per SM hide the count loop's shared-memory latency
#ifndef AUTX_RANK_THREADS
#define AUTX_RANK_THREADS 512
#endif
constexpr int RANK_THREADS = AUTX_RANK_THREADS, RANK_PER_CTA = 16, RANK_SUB = RANK_THREADS / RANK_PER_CTA;
static_assert(RANK_SUB <= 32 && (RANK_SUB & (RANK_SUB - 1)) == 0, "threads per key: a power of two, <= a warp");
__global__ void __launch_bounds__(RANK_THREADS) k_rank(Policy pol, CallTable ct, Ctl* ctl, Outputs out, KvState kv,
                                                       bool kv_on, uint32_t np) {
  pdl_wait();
  pdl_trigger();
  const uint32_t t = ctl->s_t, seqno = ctl->s_seqno;
  CHAIN_BEGIN(4);
  __shared__ uint32_t red_r[33];
  const uint32_t na = ctl->n_cand_a;
  const uint32_t n = na + ctl->n_prev;
  uint64_t* rk = reinterpret_cast<uint64_t*>(fin_smem);  // [n] keys, ~0 = no candidate
  uint64_t* ck = rk + n;                                 // [n_valid] the candidates' keys
  uint32_t* ci = reinterpret_cast<uint32_t*>(ck + n);    // [n_valid] their element index
  uint32_t* rkv = ci + n;                                // [n] kvb of each element
  uint32_t* ckv = rkv + n;                               // [n_valid] the candidates' kvb
  const bool lists = out.rank_lists != 0;
  const uint32_t e0 = blockIdx.x * RANK_PER_CTA;
  const uint32_t bnd1 = ctl->qs_bnd1;
  // (1) keys into shared memory; previous-batch keys at or before region A's boundary are region
  // A's already (self-selecting gather; bnd1 = 0 otherwise) and become sentinels.  The key loads
  // cover the buffer's capacity, so they need not wait for the counts above (one round trip).
  constexpr int RK = 8;
  const uint32_t cap = 2 * pol.max_batch;
  uint32_t nv = 0, nbv = 0;
  for (uint32_t c0 = 0; c0 < cap; c0 += RK * RANK_THREADS) {
    uint64_t kk[RK];
    uint32_t kb[RK];
#pragma unroll
    for (int r = 0; r < RK; ++r) {
      const uint32_t i = c0 + r * RANK_THREADS + threadIdx.x;
      kk[r] = i < cap ? __ldcg(out.ckey + i) : ~0ull;
      kb[r] = lists && i < cap ? __ldcg(out.ckvb + i) : 0u;
    }
#pragma unroll
    for (int r = 0; r < RK; ++r) {
      const uint32_t i = c0 + r * RANK_THREADS + threadIdx.x;
      if (i < n) {
        uint64_t k = kk[r];
        if (i >= na && (uint32_t)(k & 0x7FFFFFFFu) < bnd1) k = ~0ull;
        nv += k != ~0ull ? 1u : 0u;
        nbv += (i >= na && k != ~0ull) ? 1u : 0u;
        rk[i] = k;
        rkv[i] = kb[r];
      }
    }
  }
  // region B holds a valid key (a previous-list call of q* past region A's boundary: empty in
  // every bench workload): the general all-pairs count below; else the O(BS) bucket ranks
  const bool no_b = !__syncthreads_or(nbv != 0);
  const bool fast = no_b && out.rank_buckets;
  bool lead = false;
  uint32_t cnt = 0, eo = 0, kvs = 0, nad = 0, own_kvb = 0;
  uint64_t x = 0;
  CandRec rec;
  if (fast && e0 < na) {
    // Region A is sorted inside each of its 2K (queue, not-running) buckets (table order, or the
    // radix order), so a key's rank is sum_{q' < q} |A_q'| + its index in its bucket + its lower
    // bound in the other bucket of its queue; the kvb prefix and the admit rank follow from the
    // kvb prefix sums in bucket order and the not-running bucket sizes.  Every CTA splits the
    // <= BS keys (8 per thread) and ranks its own RANK_PER_CTA keys with one thread each.
    constexpr int IPT = MAX_BATCH / RANK_THREADS;
    constexpr int NWR = RANK_THREADS / 32;
    __shared__ uint32_t f_bcnt[32][NWR], f_boff[33], f_nr[MAX_K + 1], f_present;
    const uint32_t tid = threadIdx.x, lane = lane_id(), w = warp_id();
    const uint32_t ek = e0 + tid;
    lead = tid < RANK_PER_CTA && ek < na;
    if (lead) rec = out.cand_rec[ek];  // issued first: its latency hides behind the split
    uint64_t* s_sub = ck;   // keys in bucket order
    uint32_t* s_pos = ci;   // table index -> bucket-order position
    uint32_t* s_kvp = ckv;  // exclusive kvb prefix in bucket order, [na] = total
    if (STAMPS_ON && blockIdx.x == 0 && tid == 0) ctl->dbg[54] = globaltimer();
    if (tid == 0) f_present = 0;
    __syncthreads();
    uint32_t bk[IPT], loc[IPT], pres = 0;
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
      const uint32_t i = tid * IPT + r;
      bk[r] = 32;
      if (i < na) {
        const uint64_t k = rk[i];
        bk[r] = (uint32_t)(k >> 59) * 2u + (uint32_t)((k >> 31) & 1u);
        pres |= 1u << bk[r];
      }
    }
    pres = __reduce_or_sync(0xffffffffu, pres);
    if (lane == 0 && pres) atomicOr(&f_present, pres);
    __syncthreads();
    const uint32_t present = f_present;
    {
      const uint32_t lt = (1u << lane) - 1u;
      for (uint32_t pm = present; pm; pm &= pm - 1u) {
        const uint32_t b = __ffs(pm) - 1u;
        uint32_t below = 0, tot = 0, own = 0;
#pragma unroll
        for (int r = 0; r < IPT; ++r) {
          const uint32_t bl = __ballot_sync(0xffffffffu, bk[r] == b);
          below += __popc(bl & lt);
          tot += __popc(bl);
        }
#pragma unroll
        for (int r = 0; r < IPT; ++r)
          if (bk[r] == b) loc[r] = below + own++;
        if (lane == 0) f_bcnt[b][w] = tot;
      }
    }
    __syncthreads();
    for (uint32_t b = w; b < 32; b += NWR) {
      const bool on = (present >> b) & 1u;
      const uint32_t v = on && lane < (uint32_t)NWR ? f_bcnt[b][lane] : 0u;
      const uint32_t inc = warp_incl_scan(v);
      if (on && lane < (uint32_t)NWR) f_bcnt[b][lane] = inc - v;
      if (lane == 31) f_boff[b] = inc;  // the bucket's size, for now
    }
    __syncthreads();
    if (w == 0) {
      const uint32_t sz = f_boff[lane];
      const uint32_t inc = warp_incl_scan(sz);
      f_boff[lane] = inc - sz;
      if (lane == 31) f_boff[32] = inc;
      // not-running calls of the queues before q: the sizes of buckets 2 q' + 1, q' < q
      const uint32_t nrs = (lane & 1u) ? sz : 0u;
      const uint32_t nri = warp_incl_scan(nrs);
      if (lane & 1u) f_nr[(lane >> 1) + 1] = nri;
      if (lane == 0) f_nr[0] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
      const uint32_t i = tid * IPT + r;
      if (bk[r] < 32) {
        const uint32_t p = f_boff[bk[r]] + f_bcnt[bk[r]][w] + loc[r];
        s_sub[p] = rk[i];
        s_pos[i] = p;
        s_kvp[p] = rkv[i];
      }
    }
    __syncthreads();
    if (lists) {  // kvb prefix sums in bucket order
      uint32_t kv[IPT], sum = 0;
#pragma unroll
      for (int r = 0; r < IPT; ++r) {
        const uint32_t i = tid * IPT + r;
        kv[r] = i < na ? s_kvp[i] : 0u;
        sum += kv[r];
      }
      uint32_t tot;
      uint32_t run = block_excl_scan<uint32_t, RANK_THREADS>(sum, red_r, &tot);
#pragma unroll
      for (int r = 0; r < IPT; ++r) {
        const uint32_t i = tid * IPT + r;
        if (i < na) s_kvp[i] = run;
        run += kv[r];
      }
      if (tid == 0) s_kvp[na] = tot;
      __syncthreads();
    }
    if (STAMPS_ON && blockIdx.x == 0 && tid == 0) ctl->dbg[55] = globaltimer();
    if (blockIdx.x == 0 && tid == 0) {
      ctl->n_cand_b = 0;
      if (STAMPS_ON) { ctl->dbg[52] = na; ctl->dbg[53] = n; }
    }
    if (lead) {
      x = rk[ek];
      eo = ek;
      own_kvb = rkv[ek];
      const uint32_t q = (uint32_t)(x >> 59), nr = (uint32_t)((x >> 31) & 1u);
      const uint32_t b = 2 * q + nr, o = b ^ 1u, pos = s_pos[ek];
      const uint32_t ob = f_boff[o], on = f_boff[o + 1] - ob;
      uint32_t lb = 0;  // keys of the other bucket below x
#pragma unroll
      for (uint32_t step = (uint32_t)MAX_BATCH; step > 0; step >>= 1)
        if (lb + step <= on && s_sub[ob + lb + step - 1] < x) lb += step;
      const uint32_t idx = pos - f_boff[b];
      cnt = f_boff[2 * q] + idx + lb;
      if (lists) {
        kvs = s_kvp[f_boff[2 * q]] + (s_kvp[pos] - s_kvp[f_boff[b]]) + (s_kvp[ob + lb] - s_kvp[ob]);
        nad = f_nr[q] + (nr ? idx : lb);
      }
    }
    if (STAMPS_ON && blockIdx.x == 0 && tid == 0) ctl->dbg[56] = globaltimer();
  } else if (!fast && blockIdx.x * (RANK_PER_CTA / 2) < n) {
    // (2) compact the candidates (same deterministic order in every CTA): sentinels rank last and
    // nobody reads them, so only the n_valid candidates are ranked and compared against
    if (STAMPS_ON && blockIdx.x == 0 && threadIdx.x == 0) ctl->dbg[54] = globaltimer();
    // without region-B keys the candidates are region A, [0, na) of rk: nothing to compact
    uint32_t n_valid = na;
    const uint64_t* kp = rk;
    const uint32_t* kvp = rkv;
    if (!no_b) {
      uint32_t off = block_excl_scan<uint32_t, RANK_THREADS>(nv, red_r, &n_valid);
      for (uint32_t i = threadIdx.x; i < n; i += RANK_THREADS)
        if (rk[i] != ~0ull) { ck[off] = rk[i]; ci[off] = i; ckv[off] = rkv[i]; ++off; }
      kp = ck;
      kvp = ckv;
    }
    __syncthreads();
    if (STAMPS_ON && blockIdx.x == 0 && threadIdx.x == 0) ctl->dbg[55] = globaltimer();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctl->n_cand_b = n_valid - na;
      if (STAMPS_ON) {
        ctl->dbg[52] = n_valid;
        ctl->dbg[53] = n;
      }
    }
    // (3) rank = number of smaller keys (keys are unique), RANK_SUB threads per key; the record
    // load is issued before the count so that its latency hides behind it
    // when the candidates fill at most half the grid's capacity, a full warp per key (8 keys per
    // CTA) keeps every CTA busy and halves each thread's compares; else half a warp per key
    const bool wide = 2 * n_valid <= gridDim.x * RANK_PER_CTA && out.rank_wide;
    const uint32_t subn = wide ? 2u * RANK_SUB : (uint32_t)RANK_SUB;
    const uint32_t e = (wide ? blockIdx.x * (RANK_PER_CTA / 2) : e0) + threadIdx.x / subn, sub = threadIdx.x % subn;
    if (e < n_valid) {
      x = kp[e];
      eo = no_b ? e : ci[e];
      own_kvb = kvp[e];
      if (sub == 0) rec = eo < na ? out.cand_rec[eo] : out.prev_rec[eo - na];
      if (lists) {
        // with the rank, the kvb prefix (Alg. 1 l.34-37) and the admit rank (smaller keys of
        // calls that did not run: not resident under eager eviction)
#pragma unroll 4
        for (uint32_t j = sub; j < n_valid; j += subn) {  // (4 independent smem chains in flight)
          const uint64_t y = kp[j];
          const bool lt = y < x;
          cnt += lt ? 1u : 0u;
          kvs += lt ? kvp[j] : 0u;
          nad += (lt && ((y >> 31) & 1u)) ? 1u : 0u;
        }
      } else {
#pragma unroll 4
        for (uint32_t j = sub; j < n_valid; j += subn) cnt += kp[j] < x ? 1u : 0u;
      }
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      if ((uint32_t)d >= subn) break;
      cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
      if (lists) {
        kvs += __shfl_xor_sync(0xffffffffu, kvs, d);
        nad += __shfl_xor_sync(0xffffffffu, nad, d);
      }
    }
    if (subn > 32) {  // two warps per key: the odd warp's sums join the even warp's
      __shared__ uint32_t x_part[RANK_THREADS / 64][3];
      const uint32_t w = threadIdx.x >> 5;
      if ((w & 1u) && lane_id() == 0) { x_part[w >> 1][0] = cnt; x_part[w >> 1][1] = kvs; x_part[w >> 1][2] = nad; }
      __syncthreads();
      if (!(w & 1u)) { cnt += x_part[w >> 1][0]; kvs += x_part[w >> 1][1]; nad += x_part[w >> 1][2]; }
    }
    if (STAMPS_ON && blockIdx.x == 0 && threadIdx.x == 0) ctl->dbg[56] = globaltimer();
    lead = sub == 0 && e < n_valid;
  }
  {
    if (lead) {
      out.skey[cnt] = x;
      out.sidx[cnt] = eo;
      out.srec[cnt] = rec;
      // a resident call (previous resident-list entry rec._pad) publishes its sorted position:
      // finalize tests the previous list's membership in the new one without searching
      if (rec.qf & QF_RES) out.prev_pos[rec._pad] = (unsigned long long)seqno << 32 | cnt;
      if (lists) {
        // Alg. 1 l.32-39 for this key alone: kvb >= 1 makes the inclusive prefix strictly
        // increasing, so "count <= BS and sum kvb <= P" holds exactly on a prefix of the order
        // (the first misfit stops, R13); the batch entries write their lists and accounting
        const uint32_t incl = kvs + own_kvb;
        const uint32_t BS = pol.max_batch;
        if (cnt < BS && (pol.kv_budget == AUTX_INF || incl <= pol.kv_budget)) {
          const uint32_t sl = rec.slot;
          out.batch_slots[cnt] = sl;
          out.batch_ids[cnt] = rec.cid;
          if (out.zero_copy) { out.h_batch[cnt] = rec.cid; out.h_batch_slots[cnt] = sl; }
          // step accounting + eager demotion (Alg. 1 l.20-23)
          uint32_t q = rec.qf & QF_QMASK, qt = rec.quanta;
          ct.exec[sl] = rec.exec + 1;
          ct.mtime[sl] = rec.mtime + 1;
          if (qt != AUTX_INF) {
            qt -= 1;
            if (qt == 0) {
              q = min(q + 1, pol.K - 1);
              qt = pol.quanta[q];
            }
            ct.quanta[sl] = qt;
          }
          ct.qf[sl] = (uint8_t)(q | QF_RUN | QF_RES);
          ct.bidx[sl] = cnt;
          out.prev_slots[cnt] = sl;
          if ((x >> 31) & 1u) {  // admit: did not run in the previous step (not resident)
            out.admit_ids[nad] = rec.cid;
            out.admit_slots[nad] = sl;
            if (out.zero_copy) out.h_admit[nad] = rec.cid;
            const uint32_t held = rec.exec > 0 ? blocks_for(pol, rec.tok + rec.exec) : 0u;  // R28
            if (held) atomicAdd(&ctl->acc_swap_in, (unsigned long long)held);
            atomicMax(&ctl->acc_nadmit, nad + 1);
          }
          atomicMax(&ctl->acc_nbatch, cnt + 1);
          atomicMax(&ctl->acc_kv, (unsigned long long)incl);
        }
      }
    }
  }
  CHAIN_END(4);
}

// ---------------------------------------------------------------------------------------------
// a5 inside the finalize (AUTX_PIPELINE=ord or sel; the default keeps k_rank): the order of
// the <= 2 BS candidates in O(BS) work on one CTA, no all-pairs count.
//   Region A (the gather's candidates) is in table order, i.e. (arrival, seq) order (rows are
//   registered in arrival order, R11).  Split it into 2K sub-lists by (q, not-running): inside one
//   sub-list the key (q, arrival, not-running, seq) orders exactly as the table does, so each
//   sub-list is sorted as it stands.  A key's rank is then
//       sum_{q' < q} |A_q'|  +  its index in its own sub-list  +  lower_bound in the other
//       sub-list of its queue  (+ lower_bound in the sorted region B when q = q*).
//   Region B (previous-resident calls of q* past region A's boundary, <= BS; empty in every bench
//   workload) is sorted by a bitonic network in shared memory; a B key's rank is its index in B
//   plus its lower bounds in the two sub-lists of q*.
// Writes the first m = min(BS, |A| + |B|) keys (uk) and records (s_rec) in key order and, per
// previous-resident entry, its sorted position (s_ppos; NONE if it is no candidate).  Returns
// |B|.  pr: the previous resident list's records (finalize's preempt input), loaded here.
// ---------------------------------------------------------------------------------------------
// SEL (k_scan_emit ran instead of k_gather_ss): the selection itself is derived here.  q* is the
// first queue whose inclusive total reaches BS (the last tile's saturated inclusive prefix holds
// the totals: only whether a total reaches BS matters past the boundary), m' = BS - the totals
// before it, and region A = cq[q] for q < q* plus the first m' of cq[q*], concatenated in queue
// order (so each queue's calls stay in table order).  The previous resident list's records are
// read from the call table (its slots were loaded before the PDL wait: ps).
template <int NT, int R, bool SEL>
__device__ __forceinline__ uint32_t order_candidates(const Policy& pol, CallTable& ct, Ctl* ctl, Outputs& out,
                                                     uint32_t t, uint64_t* uk, CandRec* s_rec, uint64_t* s_sub,
                                                     uint64_t* s_bk, uint32_t* s_ppos, CandRec (&pr)[R],
                                                     const CandRec (&pp)[R], uint32_t n_prev_pre,
                                                     uint32_t& live_out, uint32_t& promo_out) {
  constexpr int NW = NT / 32;
  constexpr uint32_t FULL = 0xffffffffu;
  __shared__ uint32_t s_bcnt[32][NW];  // per (bucket, warp): items, then the warp's exclusive offset
  __shared__ uint32_t s_boff[33];      // bucket start in s_sub (bucket b = 2 q + not-running)
  __shared__ uint32_t s_present, s_nb;
  __shared__ uint32_t s_qoff[MAX_K + 1], s_sel[4];  // SEL: region A's queue offsets; nA, q*, m', bnd1
  const uint32_t tid = threadIdx.x, lane = lane_id(), w = warp_id();
  const uint32_t BS = pol.max_batch, K = pol.K;
  uint32_t nA, n_prev, bnd1, qs;
  uint64_t ka[R];
  CandRec ra[R];
  STAMP(20);
  if constexpr (SEL) {
    n_prev = n_prev_pre;
    // (1) one round: the totals, the step's counters and the previous list's records
    if (w == 0) {
      const uint32_t n_rows = ctl->s_n_rows, ntiles = n_rows ? (n_rows + TILE - 1) / TILE : 1u;
      const unsigned long long v = lane < (K + 3) / 4 ? ld_relaxed_u64(out.lb + (size_t)(ntiles - 1) * 4 + lane) : 0ull;
      uint32_t stat = lane < 2 * QP_LINES ? __ldcg(&ctl->qpart[lane >> 1][MAX_K + (lane & 1)]) : 0u;
#pragma unroll
      for (int d = 2; d < 32; d <<= 1) stat += __shfl_xor_sync(FULL, stat, d);
      const unsigned long long vq = __shfl_sync(FULL, v, (lane >> 2) & 3);
      const uint32_t tq = lane < K ? (uint32_t)(vq >> (13 * (lane & 3))) & 0x1FFFu : 0u;
      const uint32_t incl = warp_incl_scan(tq);
      const uint32_t b = __ballot_sync(FULL, lane < K && incl >= BS);
      const uint32_t q_s = b ? __ffs(b) - 1 : K;
      const uint32_t excl_s = __shfl_sync(FULL, incl - tq, q_s & 31);
      const uint32_t tot = __shfl_sync(FULL, incl, 31);
      const uint32_t m = q_s < K ? BS - excl_s : 0u;
      const uint32_t take = lane < q_s ? tq : (lane == q_s ? m : 0u);
      const uint32_t ti = warp_incl_scan(take);
      if (lane <= MAX_K) s_qoff[lane] = ti - take;
      const uint32_t live = __shfl_sync(FULL, stat, 1);  // even lanes: promotions, odd: live rows
      if (lane == 0) {
        s_sel[0] = q_s < K ? BS : tot;
        s_sel[1] = q_s;
        s_sel[2] = m;
        promo_out = stat;
        live_out = live;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (tid * R + r < n_prev) {
        // the fields the dense pass may change; the others were read before the PDL wait
        const uint32_t sl = pp[r].slot;
        pr[r] = pp[r];
        pr[r].qf = ct.qf[sl];
        pr[r].mtime = ct.mtime[sl];
        pr[r].quanta = ct.quanta[sl];
        pr[r]._pad = (pr[r].qf & QF_RES) ? pp[r]._pad : NONE;
      }
    if (tid == 0) { s_present = 0; s_nb = 0; }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (tid * R + r < n_prev) s_ppos[tid * R + r] = NONE;
    __syncthreads();
    STAMP(21);
    nA = s_sel[0];
    qs = s_sel[1];
    // (2) region A's records (dependent on the totals: one more round)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t i = tid * R + r;
      if (i < nA) {
        uint32_t q = 0;
        for (uint32_t k = 1; k < K; ++k) q = i >= s_qoff[k] ? k : q;  // offsets are non-decreasing
        ra[r] = out.cq[(size_t)q * BS + (i - s_qoff[q])];
        ka[r] = cand_key(ra[r], t);
        if (i + 1 == nA && qs < K) s_sel[3] = ra[r].slot + 1;  // region A's last q* call
      }
    }
    if (tid == 0) {
      ctl->qstar = qs;
      ctl->mprime = s_sel[2];
      ctl->n_cand_a = nA;
    }
    __syncthreads();
    bnd1 = qs < K ? s_sel[3] : 0u;
  } else {
    nA = ctl->n_cand_a; n_prev = ctl->n_prev; bnd1 = ctl->qs_bnd1; qs = ctl->qstar;
    // (1) one round of loads, unconditional below BS (the buffers hold >= BS entries)
    {
      const uint64_t* __restrict__ ck = out.ckey;
      const CandRec* __restrict__ cr = out.cand_rec;
      const CandRec* __restrict__ prc = out.prev_rec;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t i = tid * R + r;
        if (i < BS) {
          ka[r] = ck[i];
          ra[r] = cr[i];
          pr[r] = prc[i];
        }
      }
    }
    if (tid == 0) { s_present = 0; s_nb = 0; }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (tid * R + r < n_prev) s_ppos[tid * R + r] = NONE;
    __syncthreads();
  }
  uint32_t bk[R], pres = 0, nbl = 0;
  uint64_t kb[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t i = tid * R + r;
    bk[r] = 32;  // no item
    if (i < nA) {
      bk[r] = (uint32_t)(ka[r] >> 59) * 2u + (uint32_t)((ka[r] >> 31) & 1u);
      pres |= 1u << bk[r];
    }
    // region B: the gather's rule (live, queue q*, past region A's boundary slot)
    kb[r] = ~0ull;
    if (i < n_prev && !(pr[r].qf & QF_DEAD) && (pr[r].qf & QF_QMASK) == qs && pr[r].slot >= bnd1) {
      kb[r] = cand_key(pr[r], t);
      ++nbl;
    }
  }
  pres = __reduce_or_sync(FULL, pres);
  nbl = __reduce_add_sync(FULL, nbl);
  if (lane == 0) {
    if (pres) atomicOr(&s_present, pres);
    if (nbl) atomicAdd(&s_nb, nbl);
  }
  __syncthreads();
  STAMP(22);
  const uint32_t present = s_present, nB = s_nb;
  // (2) stable position inside the warp per present bucket (items ordered by (lane, r))
  uint32_t loc[R];
  {
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t pm = present; pm; pm &= pm - 1u) {
      const uint32_t b = __ffs(pm) - 1u;
      uint32_t below = 0, tot = 0, own = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t bl = __ballot_sync(FULL, bk[r] == b);
        below += __popc(bl & lt);
        tot += __popc(bl);
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (bk[r] == b) loc[r] = below + own++;
      if (lane == 0) s_bcnt[b][w] = tot;
    }
  }
  __syncthreads();
  // (3) per bucket, the warps' exclusive offsets (warp w: buckets w, w + NW, ...); then the
  // bucket starts
  for (uint32_t b = w; b < 32; b += NW) {
    const bool on = (present >> b) & 1u;
    const uint32_t v = on && lane < (uint32_t)NW ? s_bcnt[b][lane] : 0u;
    const uint32_t inc = warp_incl_scan(v);
    if (on && lane < (uint32_t)NW) s_bcnt[b][lane] = inc - v;
    if (lane == 31) s_boff[b] = inc;  // the bucket's size, for now
  }
  __syncthreads();
  if (w == 0) {
    const uint32_t sz = s_boff[lane];
    const uint32_t inc = warp_incl_scan(sz);
    s_boff[lane] = inc - sz;
    if (lane == 31) s_boff[32] = inc;
  }
  __syncthreads();
  STAMP(23);
  uint32_t idx[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    idx[r] = 0;
    if (bk[r] < 32) {
      idx[r] = s_bcnt[bk[r]][w] + loc[r];
      s_sub[s_boff[bk[r]] + idx[r]] = ka[r];
    }
  }
  // (4) region B sorted ascending (invalid entries are ~0 and sort last)
  if (nB) {
    uint32_t PB = 1;
    while (PB < n_prev) PB <<= 1;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (tid * R + r < n_prev) s_bk[tid * R + r] = kb[r];
    for (uint32_t i = n_prev + tid; i < PB; i += NT) s_bk[i] = ~0ull;
    __syncthreads();
    for (uint32_t k = 2; k <= PB; k <<= 1)
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = tid; i < PB; i += NT) {
          const uint32_t ixj = i ^ j;
          if (ixj > i) {
            const uint64_t a = s_bk[i], c = s_bk[ixj];
            if ((a > c) == ((i & k) == 0)) { s_bk[i] = c; s_bk[ixj] = a; }
          }
        }
        __syncthreads();
      }
  }
  __syncthreads();
  STAMP(24);
  // (5) ranks; the first m keys and records land in key order
  auto lower = [](const uint64_t* a, uint32_t n, uint64_t x) {  // #elements < x in sorted a[0, n)
    uint32_t lo = 0;
#pragma unroll
    for (uint32_t step = (uint32_t)MAX_BATCH; step > 0; step >>= 1)
      if (lo + step <= n && a[lo + step - 1] < x) lo += step;
    return lo;
  };
  const uint32_t m = min(BS, nA + nB);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (bk[r] < 32) {
      const uint32_t b = bk[r], o = b ^ 1u, q = b >> 1;
      uint32_t rank = s_boff[2 * q] + idx[r] + lower(s_sub + s_boff[o], s_boff[o + 1] - s_boff[o], ka[r]);
      if (nB && q == qs) rank += lower(s_bk, nB, ka[r]);
      if (rank < m) {
        uk[rank] = ka[r];
        s_rec[rank] = ra[r];
      }
      if (ra[r].qf & QF_RES) {
        AUTX_CHECK(ra[r]._pad < n_prev, "order: previous resident index", ra[r]._pad);
        s_ppos[ra[r]._pad] = rank;
      }
    }
    if (kb[r] != ~0ull) {
      const uint32_t b0 = 2 * qs;
      const uint32_t rank = s_boff[b0] + lower(s_sub + s_boff[b0], s_boff[b0 + 1] - s_boff[b0], kb[r]) +
                            lower(s_sub + s_boff[b0 + 1], s_boff[b0 + 2] - s_boff[b0 + 1], kb[r]) +
                            lower(s_bk, nB, kb[r]);
      if (rank < m) {
        uk[rank] = kb[r];
        s_rec[rank] = pr[r];
      }
      s_ppos[tid * R + r] = rank;
    }
  }
  __syncthreads();
  STAMP(25);
  return nB;
}

template <int NT, int R, bool LISTS, bool ORD, bool SEL>
__device__ void finalize_body(const Policy& pol, CallTable& ct, Ctl* ctl, Outputs& out, KvState& kv, bool kv_on,
                              uint32_t t, uint32_t np, uint32_t seqno, const CandRec (&pp)[R], uint32_t n_prev_pre) {
  uint64_t* uk = reinterpret_cast<uint64_t*>(fin_smem);    // [np] sorted keys of the first m candidates
  // admit / preempt id lists staged in shared memory for the host mirrors (16-B aligned)
  uint64_t* s_ad = uk + np;
  uint64_t* s_pr = s_ad + ((pol.max_batch + 1) & ~1u);
  // ORD (order_candidates): sorted records, region-A sub-lists, region B, previous-list positions
  CandRec* s_rec = reinterpret_cast<CandRec*>(s_pr + ((pol.max_batch + 1) & ~1u));
  uint64_t* s_sub = reinterpret_cast<uint64_t*>(s_rec + pol.max_batch);
  uint64_t* s_bk = s_sub + pol.max_batch;
  uint32_t* s_ppos = reinterpret_cast<uint32_t*>(s_bk + MAX_BATCH);
  __shared__ unsigned long long red64[33];
  __shared__ uint32_t red[33];
  __shared__ uint32_t s_nbatch;
  __shared__ unsigned long long s_kvsum;
  __shared__ HostOut s_hout;
  const uint32_t tid = threadIdx.x;
  const uint32_t BS = pol.max_batch;
  const uint32_t n_prev = ctl->n_prev;
  // region A + region B (previous-batch calls of q* not in A): no duplicates, ~0 sentinels last
  uint32_t ncand = ORD ? 0u : ctl->n_cand_a + __ldcg(&ctl->n_cand_b);
  // host-record fields, loaded with everything else in the first round
  uint32_t c_live = 0, c_promo = 0, c_err = 0, c_einfo = 0;
  // rank_lists: k_rank has written the batch and admit lists and the accounting; its totals
  constexpr bool lists = LISTS;
  uint32_t a_nb = 0, a_na = 0;
  unsigned long long a_kv = 0, a_si = 0;
  if (tid == 0) {
    c_live = ctl->n_live; c_promo = ctl->n_promoted; c_err = ctl->err; c_einfo = ctl->err_info;
    // L2 reads: with the finalize fused into k_rank's last CTA these were written in this kernel
    if (lists) {
      a_nb = __ldcg(&ctl->acc_nbatch); a_na = __ldcg(&ctl->acc_nadmit);
      a_kv = __ldcg(&ctl->acc_kv); a_si = __ldcg(&ctl->acc_swap_in);
    }
  }
  STAMP(0);
  if (tid == 0) s_nbatch = 0;
  // ---- (1) the first m = min(BS, ncand) candidates in key order: key + record, plus the
  // previous batch's records (preempt), all in one round of independent loads --------------
  uint32_t nB_ord = 0;
  CandRec pr[R];
  if constexpr (ORD) {
    uint32_t live = 0, promo = 0;
    nB_ord = order_candidates<NT, R, SEL>(pol, ct, ctl, out, t, uk, s_rec, s_sub, s_bk, s_ppos, pr, pp, n_prev_pre,
                                          live, promo);
    if (SEL && tid == 0) { c_live = live; c_promo = promo; }
    ncand = ctl->n_cand_a + nB_ord;
  }
  const uint32_t m = lists ? 0u : min(BS, ncand);
  // R items per thread, blocked (i = tid * R + r): NT * R >= BS
  uint32_t c_s[R], c_qf[R], c_tok[R], c_ex[R], c_mt[R], c_qt[R], c_kvb[R];
  uint64_t c_cid[R];
  uint32_t p_s[R], p_qf[R], p_held[R];  // previous resident list: slot, flags, blocks to swap out, key
  uint64_t p_cid[R], p_key[R];
  unsigned long long p_pos[R] = {};      // seqno << 32 | sorted position (k_rank), if use_prev_pos
  unsigned long long my_kv = 0;
  {
    // all loads of this phase first, through restrict-qualified locals, so that they overlap
    // (one L2 round trip instead of a chain of them)
    const uint64_t* __restrict__ skey = out.skey;
    const CandRec* __restrict__ srec = out.srec;
    const CandRec* __restrict__ prec = out.prev_rec;
    const unsigned long long* __restrict__ ppos = out.prev_pos;
    uint64_t kk[R];
    CandRec rc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      // unconditional below BS (buffers hold >= BS entries): the loads do not wait for the counts
      const uint32_t i = tid * R + r;
      if constexpr (ORD) {
        // order_candidates left them in shared memory (and pr in registers)
        if (i < m) { kk[r] = uk[i]; rc[r] = s_rec[i]; }
        if (i < n_prev) p_pos[r] = (unsigned long long)seqno << 32 | s_ppos[i];
      } else if (i < BS) {
        if (!lists) { kk[r] = skey[i]; rc[r] = srec[i]; }
        pr[r] = out.prev_early ? pp[r] : prec[i];
        p_pos[r] = __ldcg(ppos + i);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t i = tid * R + r;
      if (i < m) {
        uk[i] = kk[r];
        c_s[r] = rc[r].slot;
        c_qf[r] = rc[r].qf;
        c_tok[r] = rc[r].tok;
        c_ex[r] = rc[r].exec;
        c_mt[r] = rc[r].mtime;
        c_qt[r] = rc[r].quanta;
        c_cid[r] = rc[r].cid;
      }
      if (i < n_prev) {
        p_s[r] = pr[r].slot;
        p_qf[r] = pr[r].qf;
        p_cid[r] = pr[r].cid;
        p_key[r] = cand_key(pr[r], t);
        // R28: a resident call holds ceil((input + exec) / bt) blocks; one that never ran has no
        // KV content and nothing to swap out (R32: standby calls)
        p_held[r] = pr[r].exec > 0 ? blocks_for(pol, pr[r].tok + pr[r].exec) : 0u;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    c_kvb[r] = 0;
    if (tid * R + r < m) {
      c_kvb[r] = blocks_for(pol, c_tok[r] + c_ex[r] + 1);  // R14
      my_kv += c_kvb[r];
    }
  }
  STAMP(1);
  STAMP(2);
  unsigned long long kv_pre = lists ? 0ull : block_excl_scan<unsigned long long, NT>(my_kv, red64, nullptr);
  if (lists && tid == 0) s_nbatch = a_nb;
  // Alg. 1 l.34-37: take while count <= BS and sum kvb <= P; kvb >= 1 makes the prefix sums
  // strictly increasing, so the fitting items are exactly a prefix: n_batch = max fitting i + 1
  unsigned long long c_incl[R];  // inclusive kvb prefix at each item
  {
    unsigned long long incl = kv_pre;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      uint32_t i = tid * R + r;
      c_incl[r] = 0;
      if (i < m) {
        incl += c_kvb[r];
        c_incl[r] = incl;
        if (pol.kv_budget == AUTX_INF || incl <= pol.kv_budget) atomicMax(&s_nbatch, i + 1);
      }
    }
  }
  __syncthreads();
  // the resident set (R32: <= BS + X calls) and the batch, its first BS calls (n_res when X = 0)
  const uint32_t n_res = s_nbatch;
  const uint32_t n_batch = min(n_res, pol.run_batch);
  STAMP(3);
  if (tid == 0 && ncand > 0 && n_res == 0) {
    if (atomicCAS(&ctl->err, 0u, (uint32_t)AUTX_E_NOMEM) == 0u)
      ctl->err_info = (uint32_t)((lists ? out.skey[0] : uk[0]) & 0x7FFFFFFF);
  }
  // ---- (4) batch list and admit = batch calls not resident (batch order) -------------------
  unsigned long long my_ad = 0;
  if (n_res == 0 && tid == 0) s_kvsum = 0;
  if (lists && tid == 0) s_kvsum = a_kv;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    uint32_t i = tid * R + r;
    if (lists) break;  // (k_rank wrote the lists)
    if (i + 1 == n_res) s_kvsum = c_incl[r];  // sum kvb over the resident set (read after the scans below)
    if (i < n_res) {
      out.batch_slots[i] = c_s[r];
      out.batch_ids[i] = c_cid[r];
      if (!(c_qf[r] & QF_RES)) {
        uint64_t held = c_ex[r] > 0 ? blocks_for(pol, c_tok[r] + c_ex[r]) : 0;  // R28
        my_ad += (1ull << 44) | held;
      }
    }
  }
  unsigned long long ad_tot = 0;
  unsigned long long ad_pre = lists ? 0ull : block_excl_scan<unsigned long long, NT>(my_ad, red64, &ad_tot);
  if (lists) ad_tot = (unsigned long long)a_na << 44 | a_si;  // (tid 0 only: the host record)
  if (!lists) {
    uint32_t pos = (uint32_t)(ad_pre >> 44);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      uint32_t i = tid * R + r;
      if (i < n_res && !(c_qf[r] & QF_RES)) {
        out.admit_ids[pos] = c_cid[r];
        s_ad[pos] = c_cid[r];
        out.admit_slots[pos] = c_s[r];
        ++pos;
      }
    }
  }
  const uint32_t n_admit = (uint32_t)(ad_tot >> 44);
  const unsigned long long swap_in = ad_tot & ((1ull << 44) - 1);
  STAMP(4);
  // ---- (5) preempt = previous batch, still active, not in the batch (previous-batch order) ---
  unsigned long long my_pre = 0;
  uint32_t is_pre = 0;
  {
    // membership of each previous-batch row in the sorted batch prefix: fixed-length branchless
    // binary searches, the R of a thread interleaved (independent smem chains)
    uint32_t pos[R];
#pragma unroll
    for (int r = 0; r < R; ++r) pos[r] = 0;
    if (ORD || out.use_prev_pos) {
      // k_rank's sorted position of each previous-batch entry that was a candidate (entries that
      // were not, e.g. of a queue below q*, keep an older seqno and are not in the batch)
#pragma unroll
      for (int r = 0; r < R; ++r) pos[r] = (uint32_t)(p_pos[r] >> 32) == seqno ? (uint32_t)p_pos[r] : NONE;
    } else {
      for (uint32_t step = 1u << 12; step > 0; step >>= 1) {  // n_res <= 4096
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t probe = pos[r] + step;
          if (probe <= n_res && uk[probe - 1] < p_key[r]) pos[r] = probe;  // pos = #keys < key
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) pos[r] = pos[r] < n_res && uk[pos[r]] == p_key[r] ? pos[r] : NONE;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t i = tid * R + r;
      if (i < n_prev && !(p_qf[r] & QF_DEAD)) {
        const bool in = pos[r] < n_res;
        if (!in) {
          is_pre |= 1u << r;
          my_pre += (1ull << 44) | p_held[r];
        }
      }
    }
  }
  unsigned long long pre_tot;
  unsigned long long pre_pre = block_excl_scan<unsigned long long, NT>(my_pre, red64, &pre_tot);
  {
    uint32_t pos = (uint32_t)(pre_pre >> 44);
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (is_pre & (1u << r)) {
        out.preempt_ids[pos] = p_cid[r];
        s_pr[pos] = p_cid[r];
        out.preempt_slots[pos] = p_s[r];
        ct.qf[p_s[r]] = (uint8_t)(p_qf[r] & ~(QF_RUN | QF_RES));
        ++pos;
      }
  }
  const uint32_t n_preempt = (uint32_t)(pre_tot >> 44);
  const unsigned long long swap_out = pre_tot & ((1ull << 44) - 1);
  const unsigned long long kv_sum = s_kvsum;
  STAMP(5);
  STAMP(6);

  // ---- KV blocks: swap plan + allocation (a7) --------------------------------------------------
  if (kv_on) {
    // the preempt list (and its rows' flags) written above by other threads is read below
    __syncthreads();
    const uint32_t W = pol.max_blocks_per_call;
    // (1) preempted calls: host pages (size-class stacks), plan items, free GPU blocks + slots.
    // A call that never ran (R32 standby) has no KV content: its blocks are freed, not swapped.
    uint32_t base_blk = 0, base_free = 0, base_plan = 0, base_items = 0;
    const uint32_t top0 = ctl->free_top, rtop0 = ctl->rs_free_top;
    for (uint32_t c0 = 0; c0 < n_preempt; c0 += NT) {
      uint32_t i = c0 + tid;
      uint32_t s = 0, rslot = 0, nb = 0, ns = 0;
      if (i < n_preempt) {
        s = out.preempt_slots[i];
        AUTX_CHECK(!(ct.qf[s] & QF_RES), "preempt: still flagged resident", s);
        rslot = ct.loc[s];
        AUTX_CHECK(rslot < pol.max_batch, "preempt: resident slot", rslot);
        nb = kv.rs_nblk[rslot];
        AUTX_CHECK(nb == blocks_for(pol, ct.tok[s] + ct.exec[s]), "preempt: held blocks", nb * 100000 + blocks_for(pol, ct.tok[s] + ct.exec[s]));
        ns = ct.exec[s] > 0 ? nb : 0u;
      }
      uint32_t tot, ptot, itot;
      uint32_t boff = base_blk + block_excl_scan<uint32_t, NT>(nb, red, &tot);
      uint32_t poff = base_plan + block_excl_scan<uint32_t, NT>(ns, red, &ptot);
      uint32_t ioff = base_items + block_excl_scan<uint32_t, NT>(ns ? 1u : 0u, red, &itot);
      if (i < n_preempt) {
        uint32_t page = NONE, cls = 0;
        if (ns) {
          cls = ceil_log2(ns);
          // pop a page range of 2^cls pages from the class stack, else bump-allocate
          uint32_t k = atomicSub(&ctl->host_free_top[cls], 1u);
          if ((int32_t)k > 0) {
            page = kv.host_free[(size_t)cls * kv.host_free_cap + k - 1];
          } else {
            atomicAdd(&ctl->host_free_top[cls], 1u);
            page = atomicAdd(&ctl->host_bump, 1u << cls);
            if ((uint64_t)page + (1u << cls) > pol.host_pages_lo) set_err(ctl, AUTX_E_NOMEM, 1);
          }
          AUTX_CHECK(ioff < pol.max_batch && poff + ns <= kv.plan_cap, "preempt: plan", poff + ns);
          kv.plan_out[ioff] = PlanItem{page, ns, poff};
        }
        ct.loc[s] = page;
        ct.hcls[s] = cls;
        const uint32_t* src = kv.rs_blocks + (size_t)rslot * W;
        for (uint32_t j = 0; j < nb; ++j) {
          uint32_t b = src[j];
          if (j < ns) kv.plan_out_blocks[poff + j] = b;
          AUTX_CHECK(top0 + boff + j < pol.n_gpu_blocks, "preempt: free stack push", top0 + boff + j);
          kv.free_stack[top0 + boff + j] = b;
        }
        kv.rs_nblk[rslot] = 0;
      }
      uint32_t rt;
      uint32_t roff = base_free + block_excl_scan<uint32_t, NT>(i < n_preempt ? 1u : 0u, red, &rt);
      AUTX_CHECK(i >= n_preempt || rtop0 + roff < pol.max_batch, "preempt: resident-slot push", rtop0 + roff);
      if (i < n_preempt) kv.rs_free[rtop0 + roff] = rslot;
      base_blk += tot;
      base_free += rt;
      base_plan += ptot;
      base_items += itot;
    }
    __syncthreads();
    uint32_t top = top0 + base_blk, rtop = rtop0 + base_free;
    // (2) resident calls: the batch grows/allocates to kvb (the next token's block), standby
    // calls (R32) to the blocks of their existing KV; admitted calls take a resident slot
    uint32_t pop_base = 0, rs_pop = 0, in_blk = 0, in_items = 0;
    for (uint32_t c0 = 0; c0 < n_res; c0 += NT) {
      uint32_t i = c0 + tid;
      uint32_t s = 0, need = 0, have = 0, rslot = NONE, admit = 0, held = 0;
      if (i < n_res) {
        s = (uint32_t)(uk[i] & 0x7FFFFFFFu);
        uint32_t qf = ct.qf[s];
        need = ceil_div_u32(ct.tok[s] + ct.exec[s] + (i < n_batch ? 1u : 0u), pol.block_tokens);
        if (need > W) set_err(ctl, AUTX_E_NOMEM, 2);
        if (qf & QF_RES) {
          rslot = ct.loc[s];
          AUTX_CHECK(rslot < pol.max_batch, "resident: slot", rslot);
          AUTX_CHECK(kv.rs_nblk[rslot] == blocks_for(pol, ct.tok[s] + ct.exec[s]), "resident: held blocks", kv.rs_nblk[rslot]);
          have = kv.rs_nblk[rslot];
        } else {
          admit = 1;
          if (ct.exec[s] > 0) held = ceil_div_u32(ct.tok[s] + ct.exec[s], pol.block_tokens);
        }
      }
      need = max(need, have);
      uint32_t alloc = need - have;
      uint32_t tot, rt, ht, it;
      uint32_t aoff = pop_base + block_excl_scan<uint32_t, NT>(alloc, red, &tot);
      uint32_t roff = rs_pop + block_excl_scan<uint32_t, NT>(admit, red, &rt);
      uint32_t hoff = in_blk + block_excl_scan<uint32_t, NT>(held, red, &ht);
      uint32_t ioff = in_items + block_excl_scan<uint32_t, NT>(held ? 1u : 0u, red, &it);
      if (i < n_res) {
        if (admit) {
          if (roff >= rtop) set_err(ctl, AUTX_E_NOMEM, 3);
          AUTX_CHECK(roff < rtop, "admit: resident-slot pop", roff);
          rslot = kv.rs_free[rtop - 1 - roff];
          AUTX_CHECK(kv.rs_nblk[rslot] == 0, "admit: popped resident slot not empty", rslot * 100000 + kv.rs_nblk[rslot]);
        }
        AUTX_CHECK(i >= n_res || aoff + alloc <= top, "alloc: pool exhausted", aoff + alloc);
        if (aoff + alloc > top) set_err(ctl, AUTX_E_NOMEM, 4);
        AUTX_CHECK(rslot < pol.max_batch && have <= W, "alloc: slot / held", rslot);
        uint32_t* dst = kv.rs_blocks + (size_t)rslot * W;
        // pops take the blocks freed by earlier steps first (stack [0, top0)), and this step's
        // swap-outs' blocks [top0, top) only when those run out: a swap-in then never writes a
        // block this step's swap-out still reads, so the two directions can run at once
        for (uint32_t j = 0; j < alloc && have + j < W && aoff + j < top; ++j) {
          const uint32_t k = aoff + j;
          dst[have + j] = k < top0 ? kv.free_stack[top0 - 1 - k] : kv.free_stack[top - 1 - (k - top0)];
        }
        kv.rs_nblk[rslot] = need;
        if (held) {
          // swap-in: host copy -> the first `held` blocks of the new list; free host pages after
          uint32_t page = ct.loc[s];
          AUTX_CHECK(ioff < pol.max_batch && hoff + held <= kv.plan_cap && held <= W, "swap-in: plan", hoff + held);
          kv.plan_in[ioff] = PlanItem{page, held, hoff};
          for (uint32_t j = 0; j < held; ++j) kv.plan_in_blocks[hoff + j] = dst[j];
        }
        ct.loc[s] = rslot;
      }
      pop_base += tot;
      rs_pop += rt;
      in_blk += ht;
      in_items += it;
    }
    __syncthreads();
    {
      // the stack after the pops: the older blocks left, then this step's freed blocks left
      const uint32_t pops_old = min(pop_base, top0), pops_new = pop_base - pops_old;
      const uint32_t nkeep = base_blk > pops_new ? base_blk - pops_new : 0u, dst0 = top0 - pops_old;
      if (dst0 != top0) {
        for (uint32_t c0 = 0; c0 < nkeep; c0 += NT) {  // downward move, chunk by chunk (reads first)
          const uint32_t i = c0 + tid;
          const uint32_t v = i < nkeep ? kv.free_stack[top0 + i] : 0u;
          __syncthreads();
          AUTX_CHECK(i >= nkeep || top0 + i < pol.n_gpu_blocks, "free stack move", top0 + i);
          if (i < nkeep) kv.free_stack[dst0 + i] = v;
          __syncthreads();
        }
      }
      if (tid == 0) ctl->swap_serial = pops_new > 0 ? 1u : 0u;
    }
    // (3) free the host ranges of swapped-in calls (after this step's swap-out allocations)
    for (uint32_t c0 = 0; c0 < n_res; c0 += NT) {
      uint32_t i = c0 + tid;
      if (i < in_items) {
        PlanItem it = kv.plan_in[i];
        uint32_t cls = ceil_log2(it.nblk);
        uint32_t k = atomicAdd(&ctl->host_free_top[cls], 1u);
        AUTX_CHECK(k < kv.host_free_cap && cls < 32, "host range free", k);
        kv.host_free[(size_t)cls * kv.host_free_cap + k] = (uint32_t)it.host_page;
      }
    }
    // (4) block table CSR of the batch
    uint32_t b0 = 0;
    for (uint32_t c0 = 0; c0 < n_batch; c0 += NT) {
      uint32_t i = c0 + tid;
      uint32_t need = 0, rslot = 0;
      if (i < n_batch) { rslot = ct.loc[(uint32_t)(uk[i] & 0x7FFFFFFFu)]; need = kv.rs_nblk[rslot]; }
      uint32_t tot;
      uint32_t o = b0 + block_excl_scan<uint32_t, NT>(need, red, &tot);
      if (i < n_batch) {
        kv.bt_offsets[i] = o;
        const uint32_t* src = kv.rs_blocks + (size_t)rslot * W;
        for (uint32_t j = 0; j < need && o + j < kv.plan_cap; ++j) kv.bt_blocks[o + j] = src[j];
      }
      b0 += tot;
    }
    if (tid == 0) {
      kv.bt_offsets[n_batch] = b0;
      ctl->free_top = top - pop_base;
      ctl->rs_free_top = rtop - rs_pop;
      ctl->n_plan_out = base_items;
      ctl->n_plan_in = in_items;
      ctl->plan_out_chunks = base_plan;
      ctl->plan_in_chunks = in_blk;
    }
    __syncthreads();
  }

  STAMP(7);
  // ---- step accounting + eager demotion (Alg. 1 l.20-23) for the batch, from registers ------
#pragma unroll
  for (int r = 0; r < R; ++r) {
    uint32_t i = tid * R + r;
    if (!lists && i < n_batch) {
      uint32_t sl = c_s[r];
      uint32_t q = c_qf[r] & QF_QMASK, dem = c_qf[r] & QF_DEM;
      ct.exec[sl] = c_ex[r] + 1;
      ct.mtime[sl] = c_mt[r] + 1;
      uint32_t qt = c_qt[r];
      if (qt != AUTX_INF) {
        if (qt > 0) qt -= 1;
        if (qt == 0) {
          if (pol.multistep) {
            dem = QF_DEM;  // R32: demoted at the next scheduling point
          } else {
            q = min(q + 1, pol.K - 1);
            qt = pol.quanta[q];
          }
        }
        ct.quanta[sl] = qt;
      }
      ct.qf[sl] = (uint8_t)(q | dem | QF_RUN | QF_RES);
      ct.bidx[sl] = i;
      out.prev_slots[i] = sl;
    } else if (!lists && i < n_res) {
      // R32 standby: resident, not running (waits implicitly via the closed-form counters)
      const uint32_t sl = c_s[r];
      ct.qf[sl] = (uint8_t)((c_qf[r] & (QF_QMASK | QF_DEM)) | QF_RES);
      ct.bidx[sl] = i;
      out.prev_slots[i] = sl;
    }
  }
  STAMP(9);
  if (tid == 0) {
    ctl->n_prev = n_res;
    HostOut h;
    h.n_batch = n_batch;
    h.n_standby = n_res - n_batch;
    h._pad = 0;
    h.n_admit = n_admit;
    h.n_preempt = n_preempt;
    h.n_active = c_live;
    h.swap_out_blocks = swap_out;
    h.swap_in_blocks = swap_in;
    h.kv_blocks = kv_sum;
    h.n_promoted = c_promo;
    const bool may_err = kv_on || n_batch == 0;  // the only places this kernel sets an error
    h.err = may_err ? ctl->err : c_err;
    h.seqno = seqno;
    h.err_info = may_err ? ctl->err_info : c_einfo;
    ctl->n_promoted = 0;
    ctl->n_live = 0;
    ctl->qs_bnd1 = 0;
    ctl->last_n_b = ORD ? nB_ord : __ldcg(&ctl->n_cand_b);
    ctl->n_cand_b = 0;
    if (lists) { ctl->acc_nbatch = 0; ctl->acc_nadmit = 0; ctl->acc_kv = 0; ctl->acc_swap_in = 0; }
    s_hout = h;
  }
  for (uint32_t i = tid; i < QP_LINES * 32; i += NT) (&ctl->qpart[0][0])[i] = 0;
  {
    const uint32_t n_rows = ctl->s_n_rows, ntiles = n_rows ? (n_rows + TILE - 1) / TILE : 1u;
    for (uint32_t i = tid; i < (ntiles + SUP_TILES - 1) / SUP_TILES * MAX_K; i += NT) out.sup_cnt[i] = 0;
    if (SEL) {  // k_scan_emit's look-back words and ticket, for the next step's dense pass
      for (uint32_t i = tid; i < ntiles * 4; i += NT) out.lb[i] = 0;
      if (tid == 0) ctl->scan_ticket = 0;
    }
    if (tid == 0) ctl->s_tail_prev = n_rows;  // the next step's scan may read these rows early
  }
  // host-visible results: by default the device block (counts + lists) is copied out by one
  // cudaMemcpyAsync after the kernel; the zero-copy variant stores the mirrors over PCIe here
  __syncthreads();
  STAMP(10);
  if (!out.zero_copy) {
    if (tid == 0) *out.d_hout = s_hout;
  } else {
    const uint32_t nb = s_hout.n_batch + s_hout.n_standby, na = s_hout.n_admit, np_ = s_hout.n_preempt;
    // 16-B posted stores over PCIe: batch ids straight from registers (a thread's R blocked
    // items are R/2 consecutive words), admit/preempt ids from their shared-memory copies
    static_assert(R % 2 == 0, "blocked items pair into 16-B words");
#pragma unroll
    for (int k = 0; k < R / 2; ++k) {
      const uint32_t i = tid * (R / 2) + k;
      if (!lists && i < (nb + 1) / 2)
        reinterpret_cast<uint4*>(out.h_batch)[i] =
            make_uint4((uint32_t)c_cid[2 * k], (uint32_t)(c_cid[2 * k] >> 32), (uint32_t)c_cid[2 * k + 1],
                       (uint32_t)(c_cid[2 * k + 1] >> 32));
    }
    // batch slots, R consecutive u32 per thread (8- or 16-byte stores)
    if (!lists && tid * R < nb) {
      if constexpr (R == 2) reinterpret_cast<uint2*>(out.h_batch_slots)[tid] = make_uint2(c_s[0], c_s[1]);
      else if constexpr (R == 4) reinterpret_cast<uint4*>(out.h_batch_slots)[tid] = make_uint4(c_s[0], c_s[1], c_s[2], c_s[3]);
      else for (int r = 0; r < R; ++r) out.h_batch_slots[tid * R + r] = c_s[r];
    }
    const uint4* sa = reinterpret_cast<const uint4*>(s_ad);
    const uint4* sp = reinterpret_cast<const uint4*>(s_pr);
    if (!lists)
      for (uint32_t i = tid; i < (na + 1) / 2; i += NT) reinterpret_cast<uint4*>(out.h_admit)[i] = sa[i];
    for (uint32_t i = tid; i < (np_ + 1) / 2; i += NT) reinterpret_cast<uint4*>(out.h_preempt)[i] = sp[i];
    __syncthreads();
    // the host reads after the stream event that follows this kernel, which orders every store
    if (tid == 0) *out.hout = s_hout;
  }
  STAMP(8);
}

template <int NT, int R, bool LISTS = false, bool ORD = false, bool SEL = false>
__global__ void __launch_bounds__(NT) k_finalize(Policy pol, CallTable ct, Ctl* ctl, Outputs out, KvState kv,
                                                 bool kv_on, uint32_t np) {
  // SEL: the previous resident list (written by the previous finalize or compaction, both
  // complete) and its calls' fields that no kernel of this step writes (id, arrival, tokens,
  // executed steps, list index) are read while the dense pass runs
  CandRec pp[R];
  uint32_t n_prev_pre = 0;
  if (!SEL && !ORD && out.prev_early) {
    // the previous list's records come from k_gather_ss (or k_take), two kernels back: this grid
    // launched only after every k_rank CTA passed its own PDL wait, so they are complete and in L2
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (threadIdx.x * R + r < pol.max_batch) {
        const unsigned long long* q = reinterpret_cast<const unsigned long long*>(out.prev_rec + threadIdx.x * R + r);
        unsigned long long w[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) w[k] = __ldcg(q + k);
        memcpy(&pp[r], w, sizeof(CandRec));
      }
  }
  if constexpr (SEL) {
    n_prev_pre = ctl->n_prev;
    uint32_t ps[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (threadIdx.x * R + r < n_prev_pre) ps[r] = out.prev_slots[threadIdx.x * R + r];
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (threadIdx.x * R + r < n_prev_pre) {
        const uint32_t sl = ps[r];
        pp[r].slot = sl;
        pp[r].cid = ct.cid[sl];
        pp[r].arr = ct.arr[sl];
        pp[r].tok = ct.tok[sl];
        pp[r].exec = ct.exec[sl];
        pp[r]._pad = ct.bidx[sl];
      }
  }
  pdl_wait();
  pdl_trigger();
  const uint32_t t = ctl->s_t, seqno = ctl->s_seqno;
  CHAIN_BEGIN(5);
  finalize_body<NT, R, LISTS, ORD, SEL>(pol, ct, ctl, out, kv, kv_on, t, np, seqno, pp, n_prev_pre);
  if (STAMPS_ON) {
    __syncthreads();
    if (threadIdx.x == 0) {
      ctl->dbg[33 + 3 * 5] = globaltimer();
      for (int i = 0; i < 32; ++i) { ctl->dbg[64 + i] = ctl->dbg[32 + i]; ctl->dbg[32 + i] = 0; }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------------------
cudaError_t launch_complete(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl,
                            const uint32_t* slots, uint32_t n, uint32_t t, KvState kv, bool kv_on,
                            CompRec* rec_out, bool apply) {
  // size the CTA to the record count: a typical step completes ~BS/mean-decode calls
  if (n <= 32)
    return launch_pdl(k_complete<32>, 1, 32, 0, s, pol, ct, pt, ctl, slots, n, t, kv, kv_on, rec_out, apply);
  else if (n <= 256)
    return launch_pdl(k_complete<256>, 1, 256, 0, s, pol, ct, pt, ctl, slots, n, t, kv, kv_on, rec_out, apply);
  else
    return launch_pdl(k_complete<FIN_THREADS>, 1, FIN_THREADS, 0, s, pol, ct, pt, ctl, slots, n, t, kv, kv_on, rec_out, apply);
  return cudaGetLastError();
}

cudaError_t launch_apply(cudaStream_t s, const Policy& pol, ProgTable pt, const void* base,
                         uint64_t stride, uint32_t G, uint32_t t) {
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_apply<<<1, FIN_THREADS, 0, s>>>(pol, pt, (const char*)base, stride, G, t);
  return cudaGetLastError();
}

cudaError_t launch_route_hdr(cudaStream_t s, void* rec, uint64_t load, uint32_t n_comp) {
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_route_hdr<<<1, 32, 0, s>>>(reinterpret_cast<RouteHdr*>(rec), load, n_comp);
  return cudaGetLastError();
}

cudaError_t launch_route(cudaStream_t s, const void* base, uint64_t stride, uint32_t G,
                         const RouteArr* arr, uint32_t n, int8_t* pin, uint32_t threshold,
                         int32_t* out, uint32_t mode, uint32_t* rr) {
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  if (n) k_route<<<1, 32, 0, s>>>((const char*)base, stride, G, arr, n, pin, threshold, out, mode, rr);
  return cudaGetLastError();
}

cudaError_t launch_register(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt,
                            const ArrivalRec* recs, uint32_t n, uint32_t first_slot, uint32_t t,
                            const uint32_t* par) {
  if (n == 0) return cudaSuccess;
  return launch_pdl(k_register, (n + 255) / 256, 256, 0, s, pol, ct, pt, recs, n, first_slot, t, par);
  return cudaGetLastError();
}

static uint32_t pow2_at_least(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// R32 window step (multi-step scheduling): no ordering.  The candidates are the previous
// resident list (batch, then standby), in its order, without the calls that completed (the
// prologue marked them DEAD); finalize then cuts it under the KV budget exactly as a scheduling
// point's sorted candidates (the first misfit stops: lazy eviction of the tail), splits batch /
// standby and accounts.  One CTA: the list holds <= BS + X <= 2048 calls.
constexpr int WIN_THREADS = 1024;
__global__ void __launch_bounds__(WIN_THREADS) k_window(Policy pol, CallTable ct, Ctl* ctl, Outputs out) {
  __shared__ uint32_t red_w[33];
  pdl_wait();
  pdl_trigger();
  const uint32_t t = ctl->s_t, seqno = ctl->s_seqno, n_prev = ctl->n_prev;
  CHAIN_BEGIN(3);
  constexpr int R = 2;  // 2 x 1024 >= MAX_BATCH
  CandRec rc[R];
  uint32_t live[R], nl = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t j = threadIdx.x * R + r;  // blocked: the list order is kept by the scan below
    live[r] = 0;
    if (j < n_prev) {
      load_rec(ct, out.prev_slots[j], &rc[r]);
      live[r] = !(rc[r].qf & QF_DEAD);
      nl += live[r];
    }
  }
  uint32_t n_live;
  uint32_t pos = block_excl_scan<uint32_t, WIN_THREADS>(nl, red_w, &n_live);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t j = threadIdx.x * R + r;
    if (j < n_prev) {
      out.prev_rec[j] = rc[r];
      if (live[r]) {
        out.srec[pos] = rc[r];
        out.skey[pos] = cand_key(rc[r], t);  // finalize reads the slot from the low bits
        out.prev_pos[j] = (unsigned long long)seqno << 32 | pos;
        ++pos;
      }
    }
  }
  if (threadIdx.x == 0) {
    ctl->n_cand_a = n_live;
    ctl->n_cand_b = 0;
    ctl->n_live = ctl->s_n_active;
    ctl->n_promoted = 0;
    ctl->qstar = pol.K;
    ctl->mprime = 0;
  }
  CHAIN_END(3);
}

// Dynamic shared memory above 48 KB is a per-device function attribute: set for the current device
// (autx_create calls this after cudaSetDevice, once per context).
cudaError_t step_kernels_setup() {
  const int big = 200 * 1024;
  cudaError_t e = cudaFuncSetAttribute(k_finalize<FIN_THREADS, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_finalize<512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_finalize<512, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_finalize<512, 2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_finalize<FIN_THREADS, 2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_finalize<512, 2, false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_finalize<FIN_THREADS, 2, false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  return e;
}

// The step's chain on stream s, PDL-linked: [prologue (launched by the caller)] -> k_scan_tile ->
// k_gather_ss -> k_rank -> k_finalize; radix mode replaces scan + gather by the sort.
cudaError_t launch_step(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl,
                        Outputs out, KvState kv, bool kv_on, uint32_t t, uint32_t n_rows,
                        uint32_t seqno, cudaEvent_t* ev, const RadixState* rx, uint32_t arr_base,
                        uint32_t* radix_passes, bool window) {
  uint32_t ntiles = (n_rows + TILE - 1) / TILE;
  if (ntiles == 0) ntiles = 1;
  out.use_prev_pos = rx ? 0u : 1u;  // k_rank publishes previous-batch positions (select mode)
  out.prev_early = 0;               // set below for the finalize that follows k_rank
  static const bool rank_narrow = getenv("AUTX_RANK_NARROW") != nullptr;
  out.rank_wide = rank_narrow ? 0u : 1u;  // k_rank may use a warp per key when candidates are few
  // k_rank's O(BS) bucket ranks (AUTX_RANK_BUCKETS=1): parity-green, measured slower than the
  // all-pairs count spread over 128 SMs (rank span 6.4 vs 5.5 us: every CTA's redundant split costs
  // more barriers than the count it replaces)
  static const bool rank_buckets = getenv("AUTX_RANK_BUCKETS") != nullptr;
  out.rank_buckets = rank_buckets ? 1u : 0u;
  static const bool no_gprefetch = getenv("AUTX_GATHER_PREFETCH") && !strcmp(getenv("AUTX_GATHER_PREFETCH"), "0");
  if (no_gprefetch) out.gtile = nullptr;
  if (ev) cudaEventRecord(ev[0], s);
  uint32_t np = std::max<uint32_t>(pow2_at_least(2 * pol.max_batch), 2048);
  // sorted keys [np] + admit and preempt id staging [2 x even(BS)]
  const size_t fin_smem_bytes = ((size_t)np + 2 * ((pol.max_batch + 1) & ~1u)) * sizeof(uint64_t);
  static const bool fin_lists = getenv("AUTX_FINALIZE_LISTS") != nullptr;
  // R32 (standby calls, deferred demotion): the finalize decides the batch
  const bool r32 = pol.run_batch != pol.max_batch || pol.multistep;
  if (window) {
    // R32 window step: the carried resident list instead of scan, selection and ordering
    out.rank_lists = 0;
    if (ev) cudaEventRecord(ev[1], s);
    launch_pdl(k_window, 1, WIN_THREADS, 0, s, pol, ct, ctl, out);
    if (ev) cudaEventRecord(ev[2], s);
    if (pol.max_batch <= 1024)
      launch_pdl(k_finalize<512, 2>, 1, 512, fin_smem_bytes, s, pol, ct, ctl, out, kv, kv_on, np);
    else
      launch_pdl(k_finalize<FIN_THREADS, 4>, 1, FIN_THREADS, fin_smem_bytes, s, pol, ct, ctl, out, kv, kv_on, np);
    if (ev) cudaEventRecord(ev[3], s);
    return cudaGetLastError();
  }
  // default: k_scan_tile -> k_gather_ss -> k_rank -> k_finalize.  AUTX_PIPELINE=ord: the finalize
  // orders the candidates itself (no k_rank); AUTX_PIPELINE=sel: k_scan_emit -> k_finalize (no
  // gather either).  Both parity-green and measured slower on the headline.
  static const char* pipeline = getenv("AUTX_PIPELINE");
  static const bool pl_sel = pipeline && !strcmp(pipeline, "sel");
  static const bool pl_ord = pipeline && !strcmp(pipeline, "ord");
  static const bool gather_kernel = !pl_sel;
  static const bool rank_kernel = !pl_sel && !pl_ord;
  const size_t ord_smem = fin_smem_bytes + (size_t)pol.max_batch * (sizeof(CandRec) + sizeof(uint64_t) + sizeof(uint32_t)) +
                          (size_t)MAX_BATCH * sizeof(uint64_t);
  if (rx) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pol.device);
    cudaError_t e = launch_radix_order(s, pol, ct, pt, ctl, out, *rx, t, n_rows, arr_base, sms, radix_passes);
    if (e != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[1], s);
  } else if (!gather_kernel) {
    // default: the dense pass emits each queue's first BS calls and the finalize selects, orders
    // and cuts (two kernels after the prologue)
    launch_pdl(k_scan_emit, ntiles, SCAN_THREADS, 0, s, pol, ct, pt, ctl, out, 1u);
    if (ev) cudaEventRecord(ev[1], s);
    if (ev) cudaEventRecord(ev[2], s);
    out.rank_lists = 0;
    if (pol.max_batch <= 1024)
      launch_pdl(k_finalize<512, 2, false, true, true>, 1, 512, ord_smem, s, pol, ct, ctl, out, kv, kv_on, np);
    else
      launch_pdl(k_finalize<FIN_THREADS, 2, false, true, true>, 1, FIN_THREADS, ord_smem, s, pol, ct, ctl, out, kv, kv_on, np);
    if (ev) cudaEventRecord(ev[3], s);
    return cudaGetLastError();
  } else {
    // prog + L2 prefetches while the prologue runs (AUTX_SCAN_PRE, default 1: measured ~0.4 us)
    static const uint32_t pre = getenv("AUTX_SCAN_PRE") ? (uint32_t)atoi(getenv("AUTX_SCAN_PRE")) : 1u;
    launch_pdl(k_scan_tile, ntiles, SCAN_THREADS, 0, s, pol, ct, pt, ctl, out, pre);
    if (ev) cudaEventRecord(ev[1], s);
    const uint32_t ggrid = ntiles + (pol.max_batch + SCAN_THREADS - 1) / SCAN_THREADS;
    launch_pdl(k_gather_ss, ggrid, SCAN_THREADS, 0, s, pol, ct, ctl, out);
  }
  // AUTX_PIPELINE=ord: the finalize orders the candidates itself (order_candidates, O(BS) on one CTA) and
  // decides the batch; the default (and radix mode) keep the multi-CTA k_rank
  if (!rx && !rank_kernel) {
    out.rank_lists = 0;
    if (ev) cudaEventRecord(ev[2], s);
    if (pol.max_batch <= 1024)
      launch_pdl(k_finalize<512, 2, false, true>, 1, 512, ord_smem, s, pol, ct, ctl, out, kv, kv_on, np);
    else
      launch_pdl(k_finalize<FIN_THREADS, 2, false, true>, 1, FIN_THREADS, ord_smem, s, pol, ct, ctl, out, kv, kv_on, np);
    if (ev) cudaEventRecord(ev[3], s);
    return cudaGetLastError();
  }
  // k_rank also decides the batch (lists, accounting) when there is no KV allocator and its keys
  // + kvb fit shared memory; else the finalize does (AUTX_FINALIZE_LISTS forces the latter)
  out.rank_lists = (!kv_on && !rx && pol.max_batch <= 1024 && !fin_lists && !r32) ? 1u : 0u;
  // k_rank's layout: rk, ck (u64) and ci, rkv, ckv (u32) per key, 2 BS keys (rkv / ckv are
  // written even when rank_lists is off)
  size_t rank_smem = std::max<size_t>((size_t)2 * pol.max_batch * (2 * sizeof(uint64_t) + 3 * sizeof(uint32_t)),
                                      fin_smem_bytes);
  // at most one rank CTA per SM: the CTAs are dispatched while the previous kernel still holds
  // most SMs, and two packed on one SM halve each other's issue rate (measured: the count loop
  // ran 2x slower behind the self-selecting gather's grid)
  rank_smem = std::max<size_t>(rank_smem, 120 * 1024);
  const uint32_t rank_grid = (2 * pol.max_batch + RANK_PER_CTA - 1) / RANK_PER_CTA;
  if (ev) cudaEventRecord(ev[2], s);
  launch_pdl(k_rank, rank_grid, RANK_THREADS, rank_smem, s, pol, ct, ctl, out, kv, kv_on, np);
  // 512 threads x 2 candidates: 4 warps per scheduler to hide the phase's latency chains (1024
  // threads hit the 64-register cap and spill); BS > 1024 takes 1024 threads x 4
  static const bool no_prev_early = getenv("AUTX_FIN_PREV_EARLY") && !strcmp(getenv("AUTX_FIN_PREV_EARLY"), "0");
  out.prev_early = no_prev_early ? 0u : 1u;  // prev_rec is two kernels back here
  if (pol.max_batch <= 1024)
    launch_pdl(out.rank_lists ? k_finalize<512, 2, true> : k_finalize<512, 2>, 1, 512, fin_smem_bytes, s, pol, ct,
               ctl, out, kv, kv_on, np);
  else
    launch_pdl(k_finalize<FIN_THREADS, 4>, 1, FIN_THREADS, fin_smem_bytes, s, pol, ct, ctl, out, kv, kv_on, np);
  if (ev) cudaEventRecord(ev[3], s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// G8: stable compaction of the call table on the device (drop completed rows, keep (arrival, seq)
// order): live counts per 2048-row tile, then every tile scatters its live rows to their rank
// among the live rows into the other buffer of the double-buffered table and records old2new;
// one CTA remaps (and compacts) the previous resident list.  No host sort, no allocation.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(SCAN_THREADS) k_live_count(CallTable src, uint32_t n_rows, uint32_t* tile_live) {
  __shared__ uint32_t red_c[33];
  const uint32_t row0 = blockIdx.x * TILE + threadIdx.x * ROWS_PER_THREAD;
  uint32_t nl = 0;
#pragma unroll
  for (int j = 0; j < ROWS_PER_THREAD; ++j)
    nl += (row0 + j < n_rows && !(src.qf[row0 + j] & QF_DEAD)) ? 1u : 0u;
  uint32_t tot;
  block_excl_scan<uint32_t, SCAN_THREADS>(nl, red_c, &tot);
  if (threadIdx.x == 0) tile_live[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_compact(CallTable src, CallTable dst, uint32_t n_rows,
                                                          const uint32_t* tile_live, uint32_t* old2new) {
  __shared__ uint32_t red_c[33];
  const uint32_t tile = blockIdx.x, tid = threadIdx.x;
  // this tile's offset: the live rows of the tiles before it (<= a few hundred counts)
  uint32_t pre = 0;
  for (uint32_t k = tid; k < tile; k += SCAN_THREADS) pre += tile_live[k];
  uint32_t base;
  block_excl_scan<uint32_t, SCAN_THREADS>(pre, red_c, &base);
  const uint32_t row0 = tile * TILE + tid * ROWS_PER_THREAD;
  uint32_t live = 0, nl = 0;
#pragma unroll
  for (int j = 0; j < ROWS_PER_THREAD; ++j) {
    const bool l = row0 + j < n_rows && !(src.qf[row0 + j] & QF_DEAD);
    live |= l ? 1u << j : 0u;
    nl += l ? 1u : 0u;
  }
  uint32_t pos = base + block_excl_scan<uint32_t, SCAN_THREADS>(nl, red_c, nullptr);
#pragma unroll
  for (int j = 0; j < ROWS_PER_THREAD; ++j) {
    const uint32_t s = row0 + j;
    if (s >= n_rows) break;
    if (!((live >> j) & 1u)) {
      old2new[s] = NONE;
      continue;
    }
    const uint32_t i = pos++;
    old2new[s] = i;
    dst.cid[i] = src.cid[s];
    dst.prog[i] = src.prog[s];
    dst.arr[i] = src.arr[s];
    dst.qf[i] = src.qf[s];
    dst.base[i] = src.base[s];
    dst.mtime[i] = src.mtime[s];
    dst.exec[i] = src.exec[s];
    dst.quanta[i] = src.quanta[s];
    dst.inh[i] = src.inh[s];
    dst.tok[i] = src.tok[s];
    dst.loc[i] = src.loc[s];
    dst.hcls[i] = src.hcls[s];
    dst.bidx[i] = src.bidx[s];
  }
}

// The previous resident list through old2new, its completed (dropped) entries removed in order;
// the surviving entries' list index (bidx) follows.  One CTA: <= 2048 entries.
__global__ void __launch_bounds__(1024) k_remap_prev(CallTable ct, Ctl* ctl, uint32_t* prev_slots,
                                                     const uint32_t* old2new, uint32_t n_live) {
  __shared__ uint32_t red_c[33];
  const uint32_t n = ctl->n_prev;
  constexpr int R = 2;
  uint32_t v[R], nl = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t j = threadIdx.x * R + r;
    v[r] = j < n ? old2new[prev_slots[j]] : NONE;
    nl += v[r] != NONE ? 1u : 0u;
  }
  uint32_t tot;
  uint32_t pos = block_excl_scan<uint32_t, 1024>(nl, red_c, &tot);  // (reads complete before the barrier)
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (v[r] != NONE) {
      prev_slots[pos] = v[r];
      ct.bidx[v[r]] = pos;
      ++pos;
    }
  if (threadIdx.x == 0) {
    ctl->n_prev = tot;
    ctl->s_tail_prev = n_live;  // every row below n_live predates the next step's arrivals
  }
}

cudaError_t launch_compact(cudaStream_t s, CallTable src, CallTable dst, uint32_t n_rows, uint32_t n_live,
                           uint32_t* tile_live, uint32_t* old2new, Ctl* ctl, uint32_t* prev_slots) {
  const uint32_t ntiles = (n_rows + TILE - 1) / TILE;
  if (ntiles) {
    __atomic_fetch_add(&g_kernel_launches, 2ull, __ATOMIC_RELAXED);
    k_live_count<<<ntiles, SCAN_THREADS, 0, s>>>(src, n_rows, tile_live);
    k_compact<<<ntiles, SCAN_THREADS, 0, s>>>(src, dst, n_rows, tile_live, old2new);
  }
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_remap_prev<<<1, 1024, 0, s>>>(dst, ctl, prev_slots, old2new, n_live);
  return cudaGetLastError();
}

}  // namespace autx
