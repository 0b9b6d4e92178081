// sm_100a kernels of one Autellix scheduling step.  Select mode (the
// default) runs the whole step as ONE cooperative kernel, k_step:
//
//   prologue   (a1, a2)  completion records -> process table (commutative reductions), rows
//                        released; arrivals appended, inherit service, placed in a queue
//   dense pass (a3, a4)  every call: anti-starvation (integer cross-multiply) + per-tile /
//                        per-super-tile queue counts; rows the prologue touches wait for it
//   selection  (a5)      q*, m' and each tile's per-queue prefix; region A written in
//                        (queue, seq) order (a stable counting sort by queue)
//   finalize   (a5, a6, a3, a7 plan)  region B, the running-first partition inside each
//                        (queue, arrival) group, the prefix cutoff on BS and the KV budget,
//                        admit/preempt lists, step accounting and eager demotion, GPU block
//                        allocation and the swap plan, host mirrors
//
// with two in-kernel grid barriers instead of kernel boundaries.  Every step of Alg. 1 runs here;
// the host only stages records.  Citations: see autx.h.
#include <algorithm>
#include <cstdlib>

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

// Phase stamps (autx_set_timing mode 2, or always in a -DAUTX_CHAIN_STAMPS build): %globaltimer
// at the step kernel's phase boundaries into ctl->dbg[40, 56) (see k_step); the finalize moves
// them to dbg[64, 80) at the step's end.  Off by default: one uniform parameter test.
#ifdef AUTX_CHAIN_STAMPS
#define STAMPS_ON(pol) true
#else
#define STAMPS_ON(pol) ((pol).stamps != 0)
#endif

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
                              CompRec* s_rec = nullptr, const uint32_t* lin = nullptr, uint32_t* prev_qfb = nullptr) {
  __shared__ uint32_t red_u[33];
  const uint32_t tid = threadIdx.x;
  for (uint32_t base = 0; base < n; base += NT) {
    uint32_t i = base + tid;
    bool valid = i < n;
    uint32_t s = valid ? slots[i] : 0;
    CompRec r{};
    uint8_t qf0 = QF_DEAD;
    uint32_t bix = NONE;
    if (valid) {
      uint32_t e = ct.exec[s];
      qf0 = ct.qf[s];  // loaded with the record fields: one round trip
      if (prev_qfb) bix = ct.bidx[s];
      r.prog = ct.prog[s];
      r.exec = e;
      r.cp = ct.inh[s] + e;
      r.tw = (t - ct.arr[s]) - e;  // totwait: active steps arr..t-1 that did not run
      rec_out[i] = r;
      if (s_rec) s_rec[i] = r;  // the caller's shared-memory copy (n <= NT)
      if (lin) pt.crit[lin[i]] = r.cp;  // AUTX_ATLAS_EQ2: p(c) + t_c, an Eq. 2 operand
    }
    if (apply && valid) apply_record(pol, pt, r, t);
    // release the row and its KV (completed calls ran in step t-1, hence are resident)
    uint32_t nfree = 0, rslot = NONE;
    if (valid) {
      uint8_t qf = qf0;
      if (kv_on && (qf & QF_RES)) {
        rslot = ct.loc[s];
        nfree = kv.rs_nblk[rslot];
      }
      ct.qf[s] = QF_DEAD;
      ct.loc[s] = NONE;
      // a completed call ran in the previous step: its previous-batch record says it is gone
      if (prev_qfb && (qf0 & QF_RUN)) prev_qfb[bix] = QF_DEAD;
    }
    if (kv_on) {
      uint32_t tot;
      uint32_t off = block_excl_scan<uint32_t, NT>(nfree, red_u, &tot);
      uint32_t has = rslot != NONE, rtot;
      uint32_t roff = block_excl_scan<uint32_t, NT>(has, red_u, &rtot);
      uint32_t top = ctl->free_top, rtop = ctl->rs_free_top;
      if (rslot != NONE) {
        const uint32_t* src = kv.rs_blocks + (size_t)rslot * pol.max_blocks_per_call;
        for (uint32_t j = 0; j < nfree; ++j) kv.free_stack[top + off + j] = src[j];
        kv.rs_nblk[rslot] = 0;
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
}

template <int NT>
__global__ void __launch_bounds__(NT) k_complete(Policy pol, CallTable ct, ProgTable pt, Ctl* ctl,
                                                 const uint32_t* slots, uint32_t n, uint32_t t, KvState kv,
                                                 bool kv_on, CompRec* rec_out, bool apply, uint32_t* prev_qfb) {
  pdl_wait();
  pdl_trigger();
  complete_body<NT>(pol, ct, pt, ctl, slots, n, t, kv, kv_on, rec_out, apply, nullptr, nullptr, prev_qfb);
}

// Multi-engine: apply every engine's completion records (R22: sums and maxima commute, so the
// replicated tables stay identical whatever the order).  recs of rank r start at
// base + r * stride bytes, after a RouteHdr.
__global__ void __launch_bounds__(1024) k_apply(Policy pol, ProgTable pt, const char* base,
                                                       uint64_t stride, uint32_t G, uint32_t t) {
  for (uint32_t r = 0; r < G; ++r) {
    const RouteHdr* h = reinterpret_cast<const RouteHdr*>(base + r * stride);
    const CompRec* recs = reinterpret_cast<const CompRec*>(h + 1);
    const uint32_t n = h->n_comp;
    for (uint32_t i = threadIdx.x; i < n; i += 1024) apply_record(pol, pt, recs[i], t);
  }
}

// Alg. 2 over the replicated arrival batch, canonical order: tokens <= threshold -> argmin load
// (ties -> lowest engine id); else the program's pinned engine, or argmin + pin (l.5-10).  The
// chosen engine's load is incremented after each assignment (R23).  One thread: the recurrence
// through `load` is sequential by definition; G <= 8 loads stay in registers.
__global__ void k_route(const char* base, uint64_t stride, uint32_t G, const RouteArr* arr,
                        uint32_t n, int8_t* pin, uint32_t threshold, int32_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint64_t load[8];
#pragma unroll
  for (int e = 0; e < 8; ++e)
    load[e] = e < (int)G ? reinterpret_cast<const RouteHdr*>(base + e * stride)->load : ~0ull;
  for (uint32_t i = 0; i < n; ++i) {
    RouteArr a = arr[i];
    int e;
    int pinned = a.tok > threshold ? pin[a.prog] : -1;
    if (a.tok > threshold && pinned >= 0) {
      e = pinned;
    } else {
      e = 0;
      uint64_t best = load[0];
#pragma unroll
      for (int k = 1; k < 8; ++k)
        if (load[k] < best) { best = load[k]; e = k; }
      if (a.tok > threshold) pin[a.prog] = (int8_t)e;
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

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ---------------------------------------------------------------------------------------------
// Step prologue (a1 + a2) of one step: completions, then arrivals, by one CTA.  A typical step's
// records travel inside the kernel parameters (no PCIe reads), larger batches through pointers.
// Runs in the step kernel's finalize CTA (select mode) or as k_prologue (radix mode).  scratch:
// shared memory for the records (the finalize's area, unused until the prologue is over).
// ---------------------------------------------------------------------------------------------
template <int NT>
__device__ void prologue_body(const StepArgs& a, unsigned char* scratch, bool stamps = false) {
  const PrologueArgs& p = a.pro;
  const Policy& pol = a.pol;
  CallTable ct = a.ct;
  ProgTable pt = a.pt;
  KvState kv = a.kv;
  Ctl* ctl = a.ctl;
  uint32_t* s_comp = reinterpret_cast<uint32_t*>(scratch);
  ArrivalRec* s_arr = reinterpret_cast<ArrivalRec*>(scratch + PRO_INLINE * 4);
  CompRec* s_rec = reinterpret_cast<CompRec*>(scratch + PRO_INLINE * (4 + sizeof(ArrivalRec)));
  const uint32_t tid = threadIdx.x;
  const bool comp_inline = p.n_comp <= PRO_INLINE, arr_inline = p.n_arr <= PRO_INLINE;
  const bool eq2 = pol.policy == AUTX_ATLAS_EQ2;
  if (comp_inline)
    for (uint32_t i = tid; i < p.n_comp; i += NT) s_comp[i] = p.comp[i];
  if (arr_inline)
    for (uint32_t i = tid; i < p.n_arr; i += NT) s_arr[i] = p.arr[i];
  __syncthreads();
  if (comp_inline && arr_inline) {
    // typical step: arrivals inherit the service after this step's completions (R10), computed
    // here (old row value combined with the step's records of the same program, exactly what the
    // reductions leave in the row), so the row loads go out with the completion loads: one round
    uint32_t svc_old = 0;
    const bool my_arr = tid < p.n_arr;
    if (my_arr && !eq2 && !(s_arr[tid].flags & 1u)) svc_old = __ldcg(&pt.info[s_arr[tid].prog].svc);
    if (p.n_comp)
      complete_body<NT>(pol, ct, pt, ctl, s_comp, p.n_comp, p.t, kv, a.kv_on, a.rec_out, true, s_rec,
                        eq2 ? p.comp_lin : nullptr, a.out.ps.qfb);
    __syncthreads();
    if (stamps && tid == 0) ctl->dbg[57] = globaltimer();
    if (my_arr) {
      const ArrivalRec r = s_arr[tid];
      uint32_t inh = 0;
      if (eq2) {
        inh = eq2_priority(pt, p.par, r);  // parents completed this step are stored above the barrier
      } else if (!(r.flags & 1u)) {
        inh = svc_old;
        for (uint32_t i = 0; i < p.n_comp; ++i)
          if (s_rec[i].prog == r.prog) inh = pol.policy == AUTX_ATLAS ? max(inh, s_rec[i].cp) : inh + s_rec[i].exec;
      }
      register_one(pol, ct, pt, r, p.first_slot + tid, p.t, true, inh);
    }
  } else {
    if (p.n_comp)
      complete_body<NT>(pol, ct, pt, ctl, comp_inline ? s_comp : p.comp_ptr, p.n_comp, p.t, kv, a.kv_on,
                        a.rec_out, true, nullptr, eq2 ? p.comp_lin : nullptr, a.out.ps.qfb);
    // arrivals inherit the service updated by this step's completions (R10): the reductions are
    // performed at L2 before the barrier releases (fence), and register_one reads svc from L2
    if (p.n_comp && p.n_arr) __threadfence();
    __syncthreads();
    const ArrivalRec* arr = arr_inline ? s_arr : p.arr_ptr;
    for (uint32_t i = tid; i < p.n_arr; i += NT) {
      if (eq2) register_one(pol, ct, pt, arr[i], p.first_slot + i, p.t, true, eq2_priority(pt, p.par, arr[i]));
      else register_one(pol, ct, pt, arr[i], p.first_slot + i, p.t);
    }
  }
  if (tid == 0) ctl->t = p.t;
}

// Radix mode: the prologue as its own kernel, before the sort.
__global__ void __launch_bounds__(ST_THREADS) k_prologue(const __grid_constant__ StepArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  prologue_body<ST_THREADS>(a, dsm);
}

// ---------------------------------------------------------------------------------------------
// In-kernel synchronisation of the step kernel.  Its grid is launched cooperatively (every CTA is
// co-resident), so CTAs may wait for each other: a CTA barrier orders the CTA's writes before
// thread 0's gpu-scope fence and relaxed increment (a release pattern); a waiter polls with
// relaxed loads and fences once when the condition holds (an acquire pattern).  Polling with
// ld.acquire would invalidate the SM's whole L1 (CCTL.IVALL) at every poll, under the feet of the
// other CTA on the SM (measured: every phase of the step 3-5x slower).  Data written by other
// CTAs in this kernel is read with ld.cg (L2), never through L1 or the read-only path.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  const uint32_t v = ld_relaxed_u32(p);
  fence_acq_rel();
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_add_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void grid_arrive(uint32_t* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    red_relaxed_add_u32(ctr, 1u);
  }
}
__device__ __forceinline__ void grid_wait(const uint32_t* ctr, uint32_t target) {
  if (threadIdx.x == 0) {
    while (ld_relaxed_u32(ctr) < target) __nanosleep(20);
    fence_acq_rel();
  }
  __syncthreads();
}
__device__ __forceinline__ void wait_prologue(const Ctl* ctl, uint32_t seqno) {
  if (threadIdx.x == 0) {
    while (ld_relaxed_u32(&ctl->pro_seq) != seqno) __nanosleep(20);
    fence_acq_rel();
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------------
// a3 + a4: the dense pass over one thread's 8 rows.  Every live call: wait = (t - base) - mtime
// (every active step since the last reset either ran or waited), W = pwait[p] + wait,
// T = svc[p] + mtime; promote to Q_1 iff W * beta_den >= beta_num * T and not 0/0 (Alg. 1
// l.24-30, R3/R4/R7).  Demotion (l.20-23) was applied eagerly by the previous step's finalize
// (only batch calls can exhaust a quantum, and nothing in between reads q).  Bytes per call:
// qf 1 + prog 4 + base 4 + mtime 4 read; a promotion writes base (it becomes t) and only the
// fields that change: qf if q != 0, mtime if != 0, quanta if q != 0 or mtime != 0 (a call in Q_1
// that has not run since its last reset already holds Q_1's quantum).  CG: the program rows may
// have been updated in this kernel (the prologue), so they are read from L2.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t qf_at(const uint32_t (&qw)[2], int j) { return (qw[j >> 2] >> (8 * (j & 3))) & 0xffu; }
__device__ __forceinline__ uint32_t lane4(const uint4& v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }

// qw: the 8 rows' flag bytes, packed 4 per word (updated in place).
template <bool CG>
__device__ __forceinline__ void dense_rows(const Policy& pol, const CallTable& ct, const ProgTable& pt, uint32_t t,
                                           uint32_t row0, uint32_t (&qw)[2], const uint32_t (&prog)[8],
                                           uint32_t (&base)[8], uint32_t (&mtim)[8], uint64_t& hq,
                                           uint32_t& npromo, uint32_t& nlive) {
  constexpr int R = 8;
  const bool anti = pol.beta_den != 0;
  const uint32_t bnum = pol.beta_num, bden = pol.beta_den, quanta0 = pol.quanta[0];
  uint32_t svc[R], pwl[R];
  uint32_t big = t & 0x80000000u;  // any operand >= 2^31: this thread needs the exact path
  if (anti) {
#pragma unroll
    for (int j = 0; j < R; ++j) {  // the program rows of all 8 rows in one round
      const bool live = !(qf_at(qw, j) & QF_DEAD);
      const uint2* pp = reinterpret_cast<const uint2*>(&pt.info[prog[j]].pwait);
      const uint2 pw = live ? (CG ? __ldcg(pp) : __ldg(pp)) : make_uint2(0u, 0u);
      svc[j] = live ? (CG ? __ldcg(&pt.info[prog[j]].svc) : __ldg(&pt.info[prog[j]].svc)) : 0u;
      pwl[j] = pw.x;
      big |= pw.y | ((pw.x | svc[j]) & 0x80000000u);
    }
  }
  // Alg. 1 l.24-26 (R3, R4).  With t, svc and pwait below 2^31 (wait, mtime <= t), W and T
  // are below 2^32, so W * beta_den >= beta_num * T is exact as two 32x32->64 products.  A
  // warp holding any larger operand takes the 128-bit comparison (starving()) for all its rows.
  uint32_t stv = 0;  // bit j: row j starving (not 0/0 and the ratio test holds)
  if (anti) {
    if (__any_sync(__activemask(), big != 0)) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const bool live = !(qf_at(qw, j) & QF_DEAD);
        PInfo pi{0, 0, 0ull};
        if (live) {
          pi.svc = __ldcg(&pt.info[prog[j]].svc);
          pi.pwait = __ldcg(&pt.info[prog[j]].pwait);
        }
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
  bool wb = false, wm = false;
  const uint32_t qw0 = qw[0], qw1 = qw[1];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const uint32_t qf = qf_at(qw, j);
    const bool live = !(qf & QF_DEAD);
    uint32_t q = qf & QF_QMASK;
    const bool pr = live && ((stv >> j) & 1u);  // Alg. 1 l.26
    if (pr && (q | mtim[j])) ct.quanta[row0 + j] = quanta0;
    wm |= pr && mtim[j] != 0;
    wb |= pr;
    if (pr) qw[j >> 2] &= ~((uint32_t)QF_QMASK << (8 * (j & 3)));
    mtim[j] = pr ? 0u : mtim[j];
    base[j] = pr ? t : base[j];
    q = pr ? 0u : q;
    npromo += pr ? 1u : 0u;
    nlive += live ? 1u : 0u;
    hq += live ? (1ull << (4 * q)) : 0ull;
  }
  if (qw[0] != qw0 || qw[1] != qw1) *reinterpret_cast<uint2*>(ct.qf + row0) = make_uint2(qw[0], qw[1]);
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

// The dense pass over one tile (thread: 8 consecutive rows).  Rows the prologue touches wait for
// it: this step's arrivals (rows >= first_new: written by the prologue, loaded again afterwards)
// and the rows of programs with a completion in this step (s_filt: a 2048-bit filter of their
// process-table rows, built from the parameters; a collision only defers more).  Those keep the
// row fields of the first load (the prologue does not change them) and only gather their program
// rows again; the completed rows among them are known from the parameters (s_dead).  All other
// rows run at once, reading nothing the prologue writes.  qw: the rows' flags after the pass.
__device__ __forceinline__ void tile_pass(const StepArgs& a, uint32_t tile, const uint32_t* s_filt, bool filt_on,
                                          uint32_t* s_dead, uint32_t (&qw)[2], uint64_t& hq, uint32_t& npromo,
                                          uint32_t& nlive) {
  const uint32_t tid = threadIdx.x;
  const uint32_t row0 = tile * TILE + tid * ROWS_PER_THREAD;
  const bool have = row0 < a.n_rows;
  const CallTable& ct = a.ct;
  uint32_t prog[8], base[8], mtim[8];
  bool full = false, prog_only = false;
  qw[0] = qw[1] = 0x40404040u;  // QF_DEAD
  if (have) {
    const uint2 qv = *reinterpret_cast<const uint2*>(ct.qf + row0);
    const uint4 p0 = __ldcs(reinterpret_cast<const uint4*>(ct.prog + row0));
    const uint4 p1 = __ldcs(reinterpret_cast<const uint4*>(ct.prog + row0 + 4));
    const uint4 b0 = __ldcs(reinterpret_cast<const uint4*>(ct.base + row0));
    const uint4 b1 = __ldcs(reinterpret_cast<const uint4*>(ct.base + row0 + 4));
    const uint4 m0 = __ldcs(reinterpret_cast<const uint4*>(ct.mtime + row0));
    const uint4 m1 = __ldcs(reinterpret_cast<const uint4*>(ct.mtime + row0 + 4));
    qw[0] = qv.x;
    qw[1] = qv.y;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      prog[j] = lane4(j < 4 ? p0 : p1, j & 3);
      base[j] = lane4(j < 4 ? b0 : b1, j & 3);
      mtim[j] = lane4(j < 4 ? m0 : m1, j & 3);
    }
    full = a.defer_all || row0 + ROWS_PER_THREAD > a.first_new;
    if (!full && filt_on) {
#pragma unroll
      for (int j = 0; j < 8; ++j) prog_only |= ((s_filt[(prog[j] >> 5) & 63] >> (prog[j] & 31)) & 1u) != 0;
    }
    if (!full && !prog_only) dense_rows<false>(a.pol, ct, a.pt, a.t, row0, qw, prog, base, mtim, hq, npromo, nlive);
  }
  if (__syncthreads_or(full || prog_only)) {
    if (filt_on) {
      // this step's completed rows in this tile (marked dead by the prologue)
      if (tid < TILE / 32) s_dead[tid] = 0;
      __syncthreads();
      if (tid < a.pro.n_comp) {
        const uint32_t sl = a.pro.comp[tid];
        if (sl / TILE == tile) atomicOr(&s_dead[(sl % TILE) >> 5], 1u << (sl & 31));
      }
    }
    wait_prologue(a.ctl, a.seqno);
    if (full) {
      const uint2 qv = __ldcg(reinterpret_cast<const uint2*>(ct.qf + row0));
      const uint4 p0 = __ldcg(reinterpret_cast<const uint4*>(ct.prog + row0));
      const uint4 p1 = __ldcg(reinterpret_cast<const uint4*>(ct.prog + row0 + 4));
      const uint4 b0 = __ldcg(reinterpret_cast<const uint4*>(ct.base + row0));
      const uint4 b1 = __ldcg(reinterpret_cast<const uint4*>(ct.base + row0 + 4));
      const uint4 m0 = __ldcg(reinterpret_cast<const uint4*>(ct.mtime + row0));
      const uint4 m1 = __ldcg(reinterpret_cast<const uint4*>(ct.mtime + row0 + 4));
      qw[0] = qv.x;
      qw[1] = qv.y;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        prog[j] = lane4(j < 4 ? p0 : p1, j & 3);
        base[j] = lane4(j < 4 ? b0 : b1, j & 3);
        mtim[j] = lane4(j < 4 ? m0 : m1, j & 3);
      }
      dense_rows<true>(a.pol, ct, a.pt, a.t, row0, qw, prog, base, mtim, hq, npromo, nlive);
    } else if (prog_only) {
      const uint32_t dead = (s_dead[(tid * ROWS_PER_THREAD) >> 5] >> ((tid * ROWS_PER_THREAD) & 31)) & 0xFFu;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if ((dead >> j) & 1u) qw[j >> 2] = (qw[j >> 2] & ~(0xFFu << (8 * (j & 3)))) | ((uint32_t)QF_DEAD << (8 * (j & 3)));
      dense_rows<true>(a.pol, ct, a.pt, a.t, row0, qw, prog, base, mtim, hq, npromo, nlive);
    }
  }
}

// Per-tile and per-super-tile queue counts, promotions and live rows of one tile.  The 4-bit
// per-thread fields are widened to 16 bits (<= 256 per warp), two queues per word, one redux.sync
// per word of the K queues in use.
__device__ __forceinline__ void tile_publish(const StepArgs& a, uint32_t tile, uint64_t hq, uint32_t npromo,
                                             uint32_t nlive, uint32_t (*wq16)[MAX_K / 2], uint32_t* wn) {
  constexpr int NW = ST_THREADS / 32;
  const uint32_t tid = threadIdx.x, K = a.pol.K;
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
    a.out.tile_cnt[(size_t)tile * MAX_K + tid] = c;
    if (c) atomicAdd(a.out.sup_cnt + (tile / SUP_TILES) * MAX_K + tid, c);
  } else if (tid == 32) {
    uint32_t pr = 0, lv = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) { pr += wn[w] >> 16; lv += wn[w] & 0xFFFFu; }
    uint32_t* qp = a.ctl->qpart[tile % QP_LINES];
    if (pr) atomicAdd(qp + MAX_K, pr);
    if (lv) atomicAdd(qp + MAX_K + 1, lv);
  }
  __syncthreads();  // wq16 / wn reuse
}

// ---------------------------------------------------------------------------------------------
// a5 selection (after the first grid barrier).  q* = the smallest queue with
// sum_{k<=q*} total_k >= BS (K if none), m' = BS - sum_{k<q*} total_k.  The BS smallest keys
// (q, arrival, not-running, seq) are all among: every live row of a queue below q*, the first m'
// rows of q* in table order (region A), and the running rows of q* that follow them inside the
// same arrival group (region B: key order inside q* differs from table order only by moving
// running calls forward within an arrival group).  Region A is written at its position in
// (queue, seq) order: a stable counting sort by queue, base_q = sum_{k<q} total_k plus the rows
// of queue q in earlier tiles (two-level prefix: super-tiles of SUP_TILES tiles, then the earlier
// tiles of the own super-tile) plus the rank inside the tile.
// ---------------------------------------------------------------------------------------------
struct SelSmem {
  uint32_t tot[ST_THREADS / MAX_K][MAX_K];  // per group of 16 threads: partial totals
  uint32_t pre[ST_THREADS / MAX_K][MAX_K];  // ... partial prefix of the tile
  uint32_t ownk[MAX_K];                     // the tile's own counts
  uint32_t base[MAX_K], prek[MAX_K];        // sum_{k<q} total_k; rows of q in earlier tiles
  uint32_t qs, m, nx, has, n_promo, n_live;
};

__device__ void select_for(const StepArgs& a, uint32_t tile, SelSmem& S) {
  constexpr int NG = ST_THREADS / MAX_K;  // 32 groups
  const uint32_t tid = threadIdx.x, h = tid / MAX_K, k = tid % MAX_K;
  const uint32_t K = a.pol.K, BS = a.pol.max_batch;
  const uint32_t nsup = (a.ntiles + SUP_TILES - 1) / SUP_TILES;
  const bool is_tile = tile != NONE;
  const uint32_t my_sup = is_tile ? tile / SUP_TILES : 0u, tr = my_sup * SUP_TILES + h;
  uint32_t tot = 0, pre = 0;
  if (k < K) {
    // every load issued before any is consumed: the tile row, then up to 2 super-tile rows per
    // group (8M rows), more in a loop
    const bool has_tr = is_tile && h < SUP_TILES && tr <= tile;
    const uint32_t c = has_tr ? __ldcg(a.out.tile_cnt + (size_t)tr * MAX_K + k) : 0u;
    const uint32_t v0 = h < nsup ? __ldcg(a.out.sup_cnt + h * MAX_K + k) : 0u;
    const uint32_t v1 = h + NG < nsup ? __ldcg(a.out.sup_cnt + (h + NG) * MAX_K + k) : 0u;
    tot = v0 + v1;
    pre = (is_tile && h < my_sup ? v0 : 0u) + (is_tile && h + NG < my_sup ? v1 : 0u);
    for (uint32_t s = h + 2 * NG; s < nsup; s += NG) {
      const uint32_t w = __ldcg(a.out.sup_cnt + s * MAX_K + k);
      tot += w;
      pre += (is_tile && s < my_sup) ? w : 0u;
    }
    if (has_tr) {
      if (tr < tile) pre += c;
      else S.ownk[k] = c;
    }
  } else if (is_tile && h == tile % SUP_TILES) {
    S.ownk[k] = 0;
  }
  S.tot[h][k] = tot;
  S.pre[h][k] = pre;
  if (tid >= 256 && tid < 288) {
    // promotions (even lanes) and live rows (odd lanes), for the host record
    const uint32_t l = tid - 256;
    uint32_t v = __ldcg(&a.ctl->qpart[l >> 1][MAX_K + (l & 1)]);
#pragma unroll
    for (int d = 2; d < 32; d <<= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (l == 0) S.n_promo = v;
    if (l == 1) S.n_live = v;
  }
  __syncthreads();
  if (tid < 32) {
    uint32_t T = 0, P = 0, O = 0;
    if (tid < MAX_K) {
#pragma unroll 8
      for (int g = 0; g < NG; ++g) { T += S.tot[g][tid]; P += S.pre[g][tid]; }
      O = is_tile ? S.ownk[tid] : 0u;
    }
    const uint32_t incl = warp_incl_scan(T);
    const uint32_t b = __ballot_sync(0xffffffffu, tid < K && incl >= BS);
    const uint32_t qs = b ? __ffs(b) - 1 : K;
    const uint32_t base = incl - T;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t bq = __shfl_sync(0xffffffffu, base, qs & 31);
    const uint32_t m = qs < K ? BS - bq : 0u;
    const bool has = __ballot_sync(0xffffffffu, tid < K && O > 0 && (tid < qs || (tid == qs && P < m))) != 0;
    if (tid < MAX_K) {
      S.base[tid] = base;
      S.prek[tid] = P;
    }
    if (tid == 0) {
      S.qs = qs;
      S.m = m;
      S.nx = qs < K ? BS : total;
      S.has = has ? 1u : 0u;
    }
  }
  __syncthreads();
}

// Region A rows of one tile -> out.xs at their (queue, seq) positions; the tile holding the
// m'-th row of q* publishes it (region A's boundary).  Ranks inside the tile: one block scan per
// word of 4 queues (16-bit fields), over the queues <= q* (ranks: the tile has candidates).  The
// tile also writes the records of its rows that ran in the previous step to out.ps (at their
// previous-batch index), so that the finalize reads the previous batch contiguously.  The copy is
// cooperative: the owning threads only publish each row's position in shared memory, then all
// threads copy the rows in [lo, hi] with consecutive rows on consecutive lanes (coalesced loads
// from the table, coalesced stores into the struct-of-arrays records), whichever threads own them.
// sm: >= TILE * 5 + 64 bytes of shared scratch.
__device__ void extract_tile(const StepArgs& a, uint32_t tile, const uint32_t (&qw)[2], const SelSmem& S,
                             unsigned long long* red64, bool ranks, unsigned char* sm) {
  constexpr int NT = ST_THREADS;
  const uint32_t tid = threadIdx.x, K = a.pol.K;
  const uint32_t qs = S.qs, m = S.m;
  const uint32_t qmax = min(qs, K - 1);
  const uint32_t nw = ranks ? (qmax >> 2) + 1 : 0u;
  const uint32_t l0 = tid * ROWS_PER_THREAD, tile0 = tile * TILE;
  uint16_t* s_px = reinterpret_cast<uint16_t*>(sm);           // [TILE] position in region A or 0xFFFF
  uint32_t* s_qf = reinterpret_cast<uint32_t*>(sm + 2 * TILE);  // [TILE / 4] flags after the pass
  uint32_t* s_rng = reinterpret_cast<uint32_t*>(sm + 3 * TILE); // [2 * NW] per-warp lo / hi
  uint32_t pos2[4];  // positions of rows 2k, 2k+1 in 16-bit halves (BS <= 2048)
  uint32_t sel = 0, runm = 0;
  const long long et0 = clock64();
#pragma unroll
  for (int k = 0; k < 4; ++k) pos2[k] = 0xFFFFFFFFu;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t qf = qf_at(qw, j);
    runm |= (!(qf & QF_DEAD) && (qf & QF_RUN)) ? 1u << j : 0u;
  }
  for (uint32_t w = 0; w < nw; ++w) {
    uint64_t c = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t qf = qf_at(qw, j), q = qf & QF_QMASK;
      if (!(qf & QF_DEAD) && q <= qmax && (q >> 2) == w) c += 1ull << (16 * (q & 3));
    }
    uint64_t ex = block_excl_scan<unsigned long long, NT>(c, red64, nullptr);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t qf = qf_at(qw, j), q = qf & QF_QMASK;
      if (!(qf & QF_DEAD) && q <= qmax && (q >> 2) == w) {
        const uint32_t sh = 16 * (q & 3);
        const uint32_t rank = S.prek[q] + (uint32_t)((ex >> sh) & 0xFFFFu);
        ex += 1ull << sh;
        if (q < qs || rank < m) {
          sel |= 1u << j;
          const uint32_t pos = S.base[q] + rank;
          pos2[j >> 1] = (pos2[j >> 1] & ~(0xFFFFu << (16 * (j & 1)))) | (pos << (16 * (j & 1)));
          if (q == qs && rank + 1 == m) {  // region A's boundary row
            a.ctl->bnd_slot = tile0 + l0 + j;
            a.ctl->bnd_arr = __ldcg(a.ct.arr + tile0 + l0 + j);
          }
        }
      }
    }
  }
  const long long et1 = clock64();
  // publish positions and flags, and compact the rows to copy into a list (warp-aggregated
  // reservations: rows stay in order inside a warp's chunk)
  const uint32_t need = sel | runm;
  reinterpret_cast<uint4*>(s_px)[tid] = make_uint4(pos2[0], pos2[1], pos2[2], pos2[3]);
  reinterpret_cast<uint2*>(s_qf)[tid] = make_uint2(qw[0], qw[1]);
  uint16_t* s_list = reinterpret_cast<uint16_t*>(sm + 3 * TILE + 64);  // [TILE] local rows to copy
  uint32_t* s_n = s_rng;
  if (tid == 0) *s_n = 0;
  __syncthreads();
  {
    const uint32_t cnt = __popc(need);
    const uint32_t incl = warp_incl_scan(cnt);
    const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t wbase = 0;
    if (lane_id() == 31 && wtot) wbase = atomicAdd(s_n, wtot);
    wbase = __shfl_sync(0xffffffffu, wbase, 31);
    uint32_t o = wbase + incl - cnt;
    for (uint32_t nd = need; nd; nd &= nd - 1) s_list[o++] = (uint16_t)(l0 + __ffs(nd) - 1);
  }
  __syncthreads();
  const uint32_t n_copy = *s_n;
  const long long et2 = clock64();
  const CallTable& ct = a.ct;
  const RecSoA& xs = a.out.xs;
  const RecSoA& ps = a.out.ps;
  // two rows per thread per round, all loads of a round issued before any store
  for (uint32_t i0 = tid; i0 < n_copy; i0 += 2 * NT) {
    uint32_t lr[2], r[2], arr[2], tok[2], ex[2], mt[2], qt[2], bx[2];
    unsigned long long cid[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t i = i0 + u * NT;
      ok[u] = i < n_copy;
      lr[u] = ok[u] ? s_list[i] : 0u;
      r[u] = tile0 + lr[u];
      cid[u] = ok[u] ? ct.cid[r[u]] : 0ull;
      arr[u] = ok[u] ? ct.arr[r[u]] : 0u;
      tok[u] = ok[u] ? ct.tok[r[u]] : 0u;
      ex[u] = ok[u] ? ct.exec[r[u]] : 0u;
      mt[u] = ok[u] ? __ldcg(ct.mtime + r[u]) : 0u;  // (promotions of this kernel)
      qt[u] = ok[u] ? __ldcg(ct.quanta + r[u]) : 0u;
      bx[u] = ok[u] ? ct.bidx[r[u]] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!ok[u]) continue;
      const uint32_t l = lr[u];
      const uint32_t px = s_px[l];
      const uint32_t qf = (s_qf[l >> 2] >> (8 * (l & 3))) & 0xFFu;
      const bool run = !(qf & QF_DEAD) && (qf & QF_RUN);
      const uint32_t qfb = qf | (run ? bx[u] << 8 : 0u);
      if (px != 0xFFFFu) {
        xs.cid[px] = cid[u]; xs.slot[px] = r[u]; xs.arr[px] = arr[u]; xs.tok[px] = tok[u];
        xs.exec[px] = ex[u]; xs.mt[px] = mt[u]; xs.qt[px] = qt[u]; xs.qfb[px] = qfb;
      }
      if (run) {
        const uint32_t b = bx[u];
        ps.cid[b] = cid[u]; ps.slot[b] = r[u]; ps.arr[b] = arr[u]; ps.tok[b] = tok[u];
        ps.exec[b] = ex[u]; ps.mt[b] = mt[u]; ps.qt[b] = qt[u]; ps.qfb[b] = qfb;
      }
    }
  }
  if (STAMPS_ON(a.pol)) {
    __syncthreads();
    if (tid == 0) {
      atomicMax(&a.ctl->dbg[36], (unsigned long long)(et1 - et0));
      atomicMax(&a.ctl->dbg[37], (unsigned long long)(et2 - et1));
      atomicMax(&a.ctl->dbg[38], (unsigned long long)(clock64() - et2));
      atomicMax(&a.ctl->dbg[35], (unsigned long long)n_copy);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// a5 order + a6 cutoff + a3 demotion + a7 plan: one CTA of ST_THREADS, I candidates per thread
// (C = ST_THREADS * I >= 2 BS).  Y = region A ++ region B (sorted by seq) is in (queue, arrival,
// seq) order, so the key order (queue, arrival, not-running, seq) (R11, R12) is a stable
// partition of Y inside each (queue, arrival) group with the running calls first.  The batch is
// the longest prefix of that order with count <= BS and sum kvb <= P (Alg. 1 l.32-39, first
// misfit stops, R13); admit = batch calls not resident, preempt = resident calls not in the
// batch; batch calls are accounted (exec++, mtime++, quanta--; waiting calls implicitly through
// the closed-form counters) and demoted when their quantum runs out (Alg. 1 l.20-23).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ceil_log2(uint32_t x) { return x <= 1 ? 0 : 32 - __clz(x - 1); }

// exclusive max-scan over the block in thread order (0 for thread 0); smem: >= 33 words
template <int NT>
__device__ __forceinline__ uint32_t block_excl_max(uint32_t v, uint32_t* smem) {
  constexpr int NW = NT / 32;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane_id() >= (uint32_t)d) x = max(x, y);
  }
  uint32_t ex = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane_id() == 0) ex = 0;
  if (lane_id() == 31) smem[warp_id()] = x;
  __syncthreads();
  if (warp_id() == 0) {
    uint32_t w = lane_id() < NW ? smem[lane_id()] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane_id() >= (uint32_t)d) w = max(w, y);
    }
    uint32_t we = __shfl_up_sync(0xffffffffu, w, 1);
    if (lane_id() == 0) we = 0;
    if (lane_id() < NW) smem[lane_id()] = we;
  }
  __syncthreads();
  const uint32_t r = max(smem[warp_id()], ex);
  __syncthreads();
  return r;
}

template <int I>
constexpr size_t fin_smem_bytes() {
  return (size_t)ST_THREADS * I * 48 + (size_t)ST_THREADS * I / 2;
}

template <int I>
__device__ void finalize_core(const StepArgs& a, unsigned char* dsm, uint32_t qs, uint32_t mp, uint32_t nx,
                              uint32_t n_live, uint32_t n_promo, uint32_t n_prev, bool wait2,
                              unsigned long long* red64, uint32_t* red32) {
  constexpr int NT = ST_THREADS, IP = I / 2, C = NT * I;
  const Policy& pol = a.pol;
  const CallTable& ct = a.ct;
  const Outputs& out = a.out;
  const KvState& kv = a.kv;
  Ctl* ctl = a.ctl;
  uint64_t* y_cid = reinterpret_cast<uint64_t*>(dsm);
  uint32_t* y_slot = reinterpret_cast<uint32_t*>(dsm + 8 * (size_t)C);
  uint32_t* y_arr = y_slot + C;
  uint32_t* y_tok = y_arr + C;
  uint32_t* y_exec = y_tok + C;
  uint32_t* y_mt = y_exec + C;
  uint32_t* y_qt = y_mt + C;
  uint32_t* y_qfb = y_qt + C;
  uint32_t* z = y_qfb + C;    // sorted position -> index in Y
  uint32_t* hb = z + C;       // running calls before each group head; region B's slots first
  uint32_t* grun = hb + C;    // running calls up to each group's end (at the head's index)
  uint8_t* inb = reinterpret_cast<uint8_t*>(grun + C);  // previous-batch entry is in the new batch
  uint64_t* s_ad = reinterpret_cast<uint64_t*>(hb);     // admit / preempt ids for the host mirrors
  uint64_t* s_pr = reinterpret_cast<uint64_t*>(grun);   // (hb, grun are free once z is known)
  __shared__ uint32_t s_nbatch;
  __shared__ unsigned long long s_kvsum;
  __shared__ HostOut s_hout;
  const uint32_t tid = threadIdx.x, BS = pol.max_batch, K = pol.K;
  const bool stamps = STAMPS_ON(pol);
  if (wait2) grid_wait(&ctl->bar2, a.n_tile_ctas);
  if (stamps && tid == 0) ctl->dbg[44] = globaltimer();
  long long dc0 = clock64(), dc1 = 0, dc2 = 0, dc3 = 0;
  // ---- (1) one round of coalesced loads: region A, the previous batch, the boundary ------------
  uint32_t bnd_slot = 0, bnd_arr = 0;
  if (qs < K) {
    bnd_slot = __ldcg(&ctl->bnd_slot);
    bnd_arr = __ldcg(&ctl->bnd_arr);
  }
  // region A: strided (coalesced), straight into the shared-memory arrays (nx <= BS <= NT * I / 2)
  {
    const RecSoA& xs = out.xs;
    unsigned long long c[IP];
    uint32_t f[IP][7];
#pragma unroll
    for (int r = 0; r < IP; ++r) {  // every load of the round first
      const uint32_t i = min(r * NT + tid, BS - 1);
      c[r] = __ldcg(xs.cid + i);
      f[r][0] = __ldcg(xs.slot + i); f[r][1] = __ldcg(xs.arr + i); f[r][2] = __ldcg(xs.tok + i);
      f[r][3] = __ldcg(xs.exec + i); f[r][4] = __ldcg(xs.mt + i); f[r][5] = __ldcg(xs.qt + i);
      f[r][6] = __ldcg(xs.qfb + i);
    }
#pragma unroll
    for (int r = 0; r < IP; ++r) {
      const uint32_t i = r * NT + tid;
      if (i < nx) {
        y_cid[i] = c[r]; y_slot[i] = f[r][0]; y_arr[i] = f[r][1]; y_tok[i] = f[r][2];
        y_exec[i] = f[r][3]; y_mt[i] = f[r][4]; y_qt[i] = f[r][5]; y_qfb[i] = f[r][6];
      }
    }
  }
  if (stamps) { __syncthreads(); dc1 = clock64(); }
  // previous batch, blocked (preempt keeps previous-batch order): entry j = tid * IP + r
  uint32_t p_slot[IP], p_arr[IP], p_tok[IP], p_exec[IP], p_mt[IP], p_qt[IP], p_qf[IP];
  uint64_t p_cid[IP];
  {
    const RecSoA& ps = out.ps;
#pragma unroll
    for (int r = 0; r < IP; ++r) {
      const uint32_t j = min(tid * IP + r, BS - 1);
      p_cid[r] = __ldcg(ps.cid + j);
      p_slot[r] = __ldcg(ps.slot + j); p_arr[r] = __ldcg(ps.arr + j); p_tok[r] = __ldcg(ps.tok + j);
      p_exec[r] = __ldcg(ps.exec + j); p_mt[r] = __ldcg(ps.mt + j); p_qt[r] = __ldcg(ps.qt + j);
      p_qf[r] = __ldcg(ps.qfb + j) & 0xFFu;
    }
#pragma unroll
    for (int r = 0; r < IP; ++r) {
      const uint32_t j = tid * IP + r;
      if (j < n_prev) inb[j] = 0;
      else p_qf[r] = QF_DEAD;
    }
  }
  if (stamps) { __syncthreads(); dc2 = clock64(); }
  // ---- (2) region B: running calls of q* in the boundary's arrival group, past the boundary ---
  uint32_t isb = 0, nbm = 0;
#pragma unroll
  for (int r = 0; r < IP; ++r) {
    const bool b = qs < K && !(p_qf[r] & QF_DEAD) && (p_qf[r] & QF_QMASK) == qs && p_arr[r] == bnd_arr &&
                   p_slot[r] > bnd_slot;
    isb |= b ? 1u << r : 0u;
    nbm += b ? 1u : 0u;
  }
  uint32_t n_b;
  uint32_t ob = block_excl_scan<uint32_t, NT>(nbm, red32, &n_b);
  if (stamps && tid == 0) {
    dc3 = clock64();
    ctl->dbg[49] = globaltimer();
    ctl->dbg[58] = dc1 - dc0;  // clock64 cycles: region A loads
    ctl->dbg[59] = dc2 - dc1;  // previous-batch loads
    ctl->dbg[60] = dc3 - dc2;  // region-B count (block scan)
  }
#pragma unroll
  for (int r = 0; r < IP; ++r)
    if ((isb >> r) & 1u) hb[ob++] = p_slot[r];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < IP; ++r)
    if ((isb >> r) & 1u) {
      uint32_t rank = 0;
      for (uint32_t k = 0; k < n_b; ++k) rank += hb[k] < p_slot[r] ? 1u : 0u;
      const uint32_t i = nx + rank;
      y_cid[i] = p_cid[r];
      y_slot[i] = p_slot[r];
      y_arr[i] = p_arr[r];
      y_tok[i] = p_tok[r];
      y_exec[i] = p_exec[r];
      y_mt[i] = p_mt[r];
      y_qt[i] = p_qt[r];
      y_qfb[i] = p_qf[r] | ((tid * IP + r) << 8);
    }
  const uint32_t n = nx + n_b;
  __syncthreads();
  if (stamps && tid == 0) ctl->dbg[45] = globaltimer();
  // ---- (3) key order: stable partition, running calls first, inside each (queue, arrival) group.
  // Blocked items (i = tid * I + r).  For item i of the group headed at gs: rb = running items of
  // the group before i, rt = running items of the whole group (written by its last item).
  uint32_t gs[I], rex[I], runm = 0, headm = 0, my_runs = 0, my_head = 0;
#pragma unroll
  for (int r = 0; r < I; ++r) {
    const uint32_t i = tid * I + r;
    if (i < n) {
      const uint32_t qfb = y_qfb[i];
      const bool head = i == 0 || ((qfb ^ y_qfb[i - 1]) & QF_QMASK) != 0 || y_arr[i] != y_arr[i - 1];
      const bool run = (qfb & QF_RUN) != 0;
      runm |= run ? 1u << r : 0u;
      headm |= head ? 1u << r : 0u;
      my_runs += run ? 1u : 0u;
      if (head) my_head = i;
    }
  }
  const uint32_t rbase = block_excl_scan<uint32_t, NT>(my_runs, red32, nullptr);
  uint32_t cur_gs = block_excl_max<NT>(my_head, red32), cur_r = rbase;
#pragma unroll
  for (int r = 0; r < I; ++r) {
    const uint32_t i = tid * I + r;
    if (i < n) {
      if ((headm >> r) & 1u) {
        cur_gs = i;
        hb[i] = cur_r;
      }
      gs[r] = cur_gs;
      rex[r] = cur_r;
      cur_r += (runm >> r) & 1u;
      // the group's last item: the running count at its end
      const bool last = i + 1 == n || ((y_qfb[i + 1] ^ y_qfb[i]) & QF_QMASK) != 0 || y_arr[i + 1] != y_arr[i];
      if (last) grun[cur_gs] = cur_r;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < I; ++r) {
    const uint32_t i = tid * I + r;
    if (i < n) {
      const uint32_t h0 = hb[gs[r]];
      const uint32_t rb = rex[r] - h0;
      const uint32_t pos = (runm >> r) & 1u ? gs[r] + rb : gs[r] + (grun[gs[r]] - h0) + (i - gs[r] - rb);
      z[pos] = i;
    }
  }
  __syncthreads();
  if (stamps && tid == 0) ctl->dbg[50] = globaltimer();
  // ---- (4) cutoff (Alg. 1 l.34-37): kvb >= 1 makes the inclusive prefix strictly increasing,
  // so "count <= BS and sum kvb <= P" holds exactly on a prefix (n_batch = last fitting + 1) ----
  const uint32_t nc = min(n, BS);
  uint32_t kvb[I];
  unsigned long long my_kv = 0;
#pragma unroll
  for (int r = 0; r < I; ++r) {
    const uint32_t p = tid * I + r;
    kvb[r] = 0;
    if (p < nc) {
      const uint32_t i = z[p];
      kvb[r] = blocks_for(pol, y_tok[i] + y_exec[i] + 1);  // R14
      my_kv += kvb[r];
    }
  }
  if (tid == 0) s_nbatch = 0;
  unsigned long long incl = block_excl_scan<unsigned long long, NT>(my_kv, red64, nullptr);
  unsigned long long inc[I];
#pragma unroll
  for (int r = 0; r < I; ++r) {
    const uint32_t p = tid * I + r;
    incl += kvb[r];
    inc[r] = incl;
    if (p < nc && (pol.kv_budget == AUTX_INF || incl <= pol.kv_budget)) atomicMax(&s_nbatch, p + 1);
  }
  __syncthreads();
  const uint32_t n_batch = s_nbatch;
  if (tid == 0 && nc > 0 && n_batch == 0) set_err(ctl, AUTX_E_NOMEM, y_slot[z[0]]);
  if (stamps && tid == 0) ctl->dbg[46] = globaltimer();
  // ---- (5) admit = batch calls not resident (batch order; blocked for the scan) -----------------
  unsigned long long my_ad = 0;
  if (n_batch == 0 && tid == 0) s_kvsum = 0;
#pragma unroll
  for (int r = 0; r < I; ++r) {
    const uint32_t p = tid * I + r;
    if (p < n_batch) {
      const uint32_t i = z[p];
      if (p + 1 == n_batch) s_kvsum = inc[r];
      if (!(y_qfb[i] & QF_RES)) {
        const uint32_t e = y_exec[i];
        const uint64_t held = e > 0 ? blocks_for(pol, y_tok[i] + e) : 0u;  // R28
        my_ad += (1ull << 44) | held;
      }
    }
  }
  unsigned long long ad_tot;
  const unsigned long long ad_pre = block_excl_scan<unsigned long long, NT>(my_ad, red64, &ad_tot);
  {
    uint32_t pos = (uint32_t)(ad_pre >> 44);
#pragma unroll
    for (int r = 0; r < I; ++r) {
      const uint32_t p = tid * I + r;
      if (p < n_batch) {
        const uint32_t i = z[p];
        if (!(y_qfb[i] & QF_RES)) {
          out.admit_ids[pos] = y_cid[i];
          out.admit_slots[pos] = y_slot[i];
          s_ad[pos] = y_cid[i];
          ++pos;
        }
      }
    }
  }
  const uint32_t n_admit = (uint32_t)(ad_tot >> 44);
  const unsigned long long swap_in = ad_tot & ((1ull << 44) - 1);
  // batch list (strided: coalesced stores) and the previous batch's membership marks
#pragma unroll
  for (int r = 0; r < I; ++r) {
    const uint32_t p = r * NT + tid;
    if (p < n_batch) {
      const uint32_t i = z[p];
      const uint32_t qfb = y_qfb[i];
      out.batch_slots[p] = y_slot[i];
      out.batch_ids[p] = y_cid[i];
      if (qfb & QF_RUN) inb[qfb >> 8] = 1;
    }
  }
  __syncthreads();
  if (stamps && tid == 0) ctl->dbg[51] = globaltimer();
  // ---- (6) preempt = previous batch, still active, not in the batch (previous-batch order) ---
  unsigned long long my_pre = 0;
  uint32_t is_pre = 0;
#pragma unroll
  for (int r = 0; r < IP; ++r) {
    const uint32_t j = tid * IP + r;
    if (j < n_prev && !(p_qf[r] & QF_DEAD) && !inb[j]) {
      is_pre |= 1u << r;
      my_pre += (1ull << 44) | blocks_for(pol, p_tok[r] + p_exec[r]);  // R28: held = ceil((tok + exec) / bt)
    }
  }
  unsigned long long pre_tot;
  const unsigned long long pre_pre = block_excl_scan<unsigned long long, NT>(my_pre, red64, &pre_tot);
  {
    uint32_t pos = (uint32_t)(pre_pre >> 44);
#pragma unroll
    for (int r = 0; r < IP; ++r)
      if ((is_pre >> r) & 1u) {
        out.preempt_ids[pos] = p_cid[r];
        s_pr[pos] = p_cid[r];
        out.preempt_slots[pos] = p_slot[r];
        ct.qf[p_slot[r]] = (uint8_t)(p_qf[r] & ~(QF_RUN | QF_RES | QF_INB));
        ++pos;
      }
  }
  const uint32_t n_preempt = (uint32_t)(pre_tot >> 44);
  const unsigned long long swap_out = pre_tot & ((1ull << 44) - 1);
  if (stamps && tid == 0) ctl->dbg[52] = globaltimer();
  // ---- (7) KV blocks: swap plan + allocation (a7) ---------------------------------------------
  if (a.kv_on) {
    __syncthreads();  // preempt_slots
    const uint32_t W = pol.max_blocks_per_call;
    // (7a) preempted calls: host pages (size-class stacks), plan items, free GPU blocks + slots
    uint32_t base_blk = 0, base_free = 0;
    const uint32_t top0 = ctl->free_top, rtop0 = ctl->rs_free_top;
    for (uint32_t c0 = 0; c0 < n_preempt; c0 += NT) {
      const uint32_t i = c0 + tid;
      uint32_t s = 0, rslot = 0, nb = 0;
      if (i < n_preempt) {
        s = out.preempt_slots[i];
        rslot = ct.loc[s];
        nb = kv.rs_nblk[rslot];
      }
      uint32_t tot;
      uint32_t boff = base_blk + block_excl_scan<uint32_t, NT>(nb, red32, &tot);
      if (i < n_preempt) {
        const uint32_t cls = ceil_log2(nb);
        // pop a page range of 2^cls pages from the class stack, else bump-allocate
        uint32_t page;
        const uint32_t k = atomicSub(&ctl->host_free_top[cls], 1u);
        if ((int32_t)k > 0) {
          page = kv.host_free[(size_t)cls * kv.host_free_cap + k - 1];
        } else {
          atomicAdd(&ctl->host_free_top[cls], 1u);
          page = atomicAdd(&ctl->host_bump, 1u << cls);
          if ((uint64_t)page + (1u << cls) > pol.host_pages_lo) set_err(ctl, AUTX_E_NOMEM, 1);
        }
        ct.loc[s] = page;
        ct.hcls[s] = cls;
        kv.plan_out[i] = PlanItem{page, nb, boff};
        const uint32_t* src = kv.rs_blocks + (size_t)rslot * W;
        for (uint32_t j = 0; j < nb; ++j) {
          const uint32_t b = src[j];
          kv.plan_out_blocks[boff + j] = b;
          kv.free_stack[top0 + boff + j] = b;
        }
        kv.rs_nblk[rslot] = 0;
      }
      uint32_t rt;
      const uint32_t roff = base_free + block_excl_scan<uint32_t, NT>(i < n_preempt ? 1u : 0u, red32, &rt);
      if (i < n_preempt) kv.rs_free[rtop0 + roff] = rslot;
      base_blk += tot;
      base_free += rt;
    }
    __syncthreads();
    const uint32_t top = top0 + base_blk, rtop = rtop0 + base_free;
    // (7b) batch calls: grow/allocate to kvb; admitted calls take a resident slot
    uint32_t pop_base = 0, rs_pop = 0, in_blk = 0, in_items = 0;
    for (uint32_t c0 = 0; c0 < n_batch; c0 += NT) {
      const uint32_t i = c0 + tid;
      uint32_t s = 0, need = 0, have = 0, rslot = NONE, admit = 0, held = 0;
      if (i < n_batch) {
        s = y_slot[z[i]];
        const uint32_t qf = ct.qf[s];
        need = ceil_div_u32(ct.tok[s] + ct.exec[s] + 1, pol.block_tokens);
        if (need > W) set_err(ctl, AUTX_E_NOMEM, 2);
        if (qf & QF_RES) {
          rslot = ct.loc[s];
          have = kv.rs_nblk[rslot];
        } else {
          admit = 1;
          if (ct.exec[s] > 0) held = ceil_div_u32(ct.tok[s] + ct.exec[s], pol.block_tokens);
        }
      }
      const uint32_t alloc = need > have ? need - have : 0;
      uint32_t tot, rt, ht, it;
      const uint32_t aoff = pop_base + block_excl_scan<uint32_t, NT>(alloc, red32, &tot);
      const uint32_t roff = rs_pop + block_excl_scan<uint32_t, NT>(admit, red32, &rt);
      const uint32_t hoff = in_blk + block_excl_scan<uint32_t, NT>(held, red32, &ht);
      const uint32_t ioff = in_items + block_excl_scan<uint32_t, NT>(held ? 1u : 0u, red32, &it);
      if (i < n_batch) {
        if (admit) {
          if (roff >= rtop) set_err(ctl, AUTX_E_NOMEM, 3);
          rslot = kv.rs_free[rtop - 1 - roff];
        }
        if (aoff + alloc > top) set_err(ctl, AUTX_E_NOMEM, 4);
        uint32_t* dst = kv.rs_blocks + (size_t)rslot * W;
        for (uint32_t j = 0; j < alloc && have + j < W && aoff + j < top; ++j)
          dst[have + j] = kv.free_stack[top - 1 - aoff - j];
        kv.rs_nblk[rslot] = need;
        if (held) {
          // swap-in: host copy -> the first `held` blocks of the new list; free host pages after
          const uint32_t page = ct.loc[s];
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
    // (7c) free the host ranges of swapped-in calls (after this step's swap-out allocations)
    for (uint32_t c0 = 0; c0 < n_batch; c0 += NT) {
      const uint32_t i = c0 + tid;
      if (i < in_items) {
        const PlanItem itm = kv.plan_in[i];
        const uint32_t cls = ceil_log2(itm.nblk);
        const uint32_t k = atomicAdd(&ctl->host_free_top[cls], 1u);
        kv.host_free[(size_t)cls * kv.host_free_cap + k] = (uint32_t)itm.host_page;
      }
    }
    // (7d) block table CSR of the batch
    uint32_t b0 = 0;
    for (uint32_t c0 = 0; c0 < n_batch; c0 += NT) {
      const uint32_t i = c0 + tid;
      uint32_t need = 0, rslot = 0;
      if (i < n_batch) {
        rslot = ct.loc[y_slot[z[i]]];
        need = kv.rs_nblk[rslot];
      }
      uint32_t tot;
      const uint32_t o = b0 + block_excl_scan<uint32_t, NT>(need, red32, &tot);
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
      ctl->n_plan_out = n_preempt;
      ctl->n_plan_in = in_items;
      ctl->plan_out_chunks = base_blk;
      ctl->plan_in_chunks = in_blk;
    }
    __syncthreads();
  }
  // ---- (8) step accounting + eager demotion (Alg. 1 l.20-23) for the batch (strided: the
  // batch is nearly in table order, so neighbouring threads write neighbouring rows) ------------
#pragma unroll
  for (int r = 0; r < I; ++r) {
    const uint32_t p = r * NT + tid;
    if (p < n_batch) {
      const uint32_t i = z[p];
      const uint32_t sl = y_slot[i];
      uint32_t q = y_qfb[i] & QF_QMASK, qt = y_qt[i];
      ct.exec[sl] = y_exec[i] + 1;
      ct.mtime[sl] = y_mt[i] + 1;
      if (qt != AUTX_INF) {
        qt -= 1;
        if (qt == 0) {
          q = min(q + 1, K - 1);
          qt = pol.quanta[q];
        }
        ct.quanta[sl] = qt;
      }
      ct.qf[sl] = (uint8_t)(q | QF_RUN | QF_RES);
      ct.bidx[sl] = p;
      out.prev_slots[p] = sl;
    }
  }
  if (stamps) {
    __syncthreads();
    if (tid == 0) ctl->dbg[53] = globaltimer();
  }
  // ---- (9) host record, host mirrors, counters reset for the next step ------------------------
  if (tid == 0) {
    ctl->n_prev = n_batch;
    ctl->qstar = qs;
    ctl->mprime = mp;
    ctl->n_x = nx;
    ctl->n_b = n_b;
    HostOut h;
    h.n_batch = n_batch;
    h.n_admit = n_admit;
    h.n_preempt = n_preempt;
    h.n_active = n_live;
    h.swap_out_blocks = swap_out;
    h.swap_in_blocks = swap_in;
    h.kv_blocks = n_batch ? s_kvsum : 0ull;
    h.n_promoted = n_promo;
    h.err = ctl->err;
    h.seqno = a.seqno;
    h.err_info = ctl->err_info;
    ctl->n_promoted = 0;
    ctl->n_live = 0;
    ctl->bar1 = 0;
    ctl->bar2 = 0;
    s_hout = h;
  }
  for (uint32_t i = tid; i < QP_LINES * 32; i += NT) (&ctl->qpart[0][0])[i] = 0;
  for (uint32_t i = tid; i < out.n_sup * MAX_K; i += NT) out.sup_cnt[i] = 0;
  __syncthreads();
  if (!out.zero_copy) {
    if (tid == 0) *out.d_hout = s_hout;
  } else {
    // 16-B posted stores over PCIe: pairs of batch ids, groups of 4 slots, admit/preempt ids from
    // their shared-memory copies
    const uint32_t nb = n_batch;
    for (uint32_t k = tid; k < (nb + 1) / 2; k += NT) {
      const uint64_t c0 = y_cid[z[2 * k]], c1 = 2 * k + 1 < nb ? y_cid[z[2 * k + 1]] : 0ull;
      reinterpret_cast<uint4*>(out.h_batch)[k] = make_uint4((uint32_t)c0, (uint32_t)(c0 >> 32), (uint32_t)c1, (uint32_t)(c1 >> 32));
    }
    for (uint32_t k = tid; k < (nb + 3) / 4; k += NT) {
      uint32_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = 4 * k + u < nb ? y_slot[z[4 * k + u]] : 0u;
      reinterpret_cast<uint4*>(out.h_batch_slots)[k] = make_uint4(v[0], v[1], v[2], v[3]);
    }
    const uint4* sa = reinterpret_cast<const uint4*>(s_ad);
    const uint4* sp = reinterpret_cast<const uint4*>(s_pr);
    for (uint32_t i = tid; i < (n_admit + 1) / 2; i += NT) reinterpret_cast<uint4*>(out.h_admit)[i] = sa[i];
    for (uint32_t i = tid; i < (n_preempt + 1) / 2; i += NT) reinterpret_cast<uint4*>(out.h_preempt)[i] = sp[i];
    __syncthreads();
    // the host reads after the stream event that follows this kernel, which orders every store
    if (tid == 0) *out.hout = s_hout;
  }
  if (stamps && tid == 0) {
    ctl->dbg[47] = globaltimer();
    for (int i = 0; i < 24; ++i) {
      ctl->dbg[64 + i] = ctl->dbg[40 + i];
      ctl->dbg[40 + i] = 0;
    }
    ctl->dbg[88] = ctl->dbg[39];
    ctl->dbg[89] = ctl->dbg[36];
    ctl->dbg[90] = ctl->dbg[37];
    ctl->dbg[91] = ctl->dbg[38];
    ctl->dbg[92] = ctl->dbg[35];
    ctl->dbg[39] = ctl->dbg[36] = ctl->dbg[37] = ctl->dbg[38] = ctl->dbg[35] = 0;
    ctl->dbg[40] = ~0ull;
  }
}

// ---------------------------------------------------------------------------------------------
// The step kernel (select mode): one cooperative launch per step.
//   CTAs 0 .. n_tile_ctas-1: the dense pass over their tiles (a3, a4) with per-queue counts;
//     grid barrier 1; selection and region-A extraction (a5); arrive at barrier 2.
//   CTA n_tile_ctas: the prologue (a1, a2: completions and arrivals), the "prologue done" flag
//     the deferred rows wait for; barrier 1; selection; the previous batch's slots; barrier 2;
//     order, cutoff, lists, accounting, KV plan (a5, a6, a3, a7).
// Stamps (dbg): 40 first CTA start, 41 last CTA start, 42 prologue done, 43 barrier 1 passed,
// 44 barrier 2 passed, 45 region B placed, 46 cutoff, 47 end, 48 last tile CTA at barrier 1,
// 49 finalize loads consumed, 50 key order, 51 batch + admit lists, 52 preempt list,
// 53 accounting (+ KV plan), 54 / 55 tile 0 selection / extraction done, 56 last tile CTA at
// barrier 2, 57 prologue completions applied.
// ---------------------------------------------------------------------------------------------
template <int I>
__global__ void __launch_bounds__(ST_THREADS, 2) k_step(const __grid_constant__ StepArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ SelSmem S;
  __shared__ unsigned long long red64[33];
  __shared__ uint32_t red32[33];
  __shared__ uint32_t wq16[ST_THREADS / 32][MAX_K / 2];
  __shared__ uint32_t wn[ST_THREADS / 32];
  const uint32_t tid = threadIdx.x;
  Ctl* ctl = a.ctl;
  const bool stamps = STAMPS_ON(a.pol);
  if (stamps && tid == 0) {
    const unsigned long long g = globaltimer();
    atomicMin(&ctl->dbg[40], g);
    atomicMax(&ctl->dbg[41], g);
  }
  if (blockIdx.x == a.n_tile_ctas) {
    // ---- prologue + finalize CTA ----
    if (a.pro_first) {
      // the prologue's rows into L2 ahead of the tiles' stream (it is on the critical path: the
      // deferred rows wait for it), then let the tiles go
      const PrologueArgs& p = a.pro;
      if (tid < p.n_comp && p.n_comp <= PRO_INLINE) {
        const uint32_t sl = p.comp[tid];
        prefetch_l2(a.ct.exec + sl); prefetch_l2(a.ct.qf + sl); prefetch_l2(a.ct.prog + sl);
        prefetch_l2(a.ct.inh + sl); prefetch_l2(a.ct.arr + sl); prefetch_l2(a.ct.bidx + sl);
        prefetch_l2(a.ct.loc + sl); prefetch_l2(a.pt.info + p.comp_prog[tid]);
      }
      if (tid < p.n_arr && p.n_arr <= PRO_INLINE) prefetch_l2(a.pt.info + p.arr[tid].prog);
      __syncthreads();
      if (tid == 0) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(&ctl->go_seq), "r"(a.seqno) : "memory");
    }
    if (a.do_pro) prologue_body<ST_THREADS>(a, dsm, stamps);
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_u32(&ctl->pro_seq, a.seqno);
      if (stamps) ctl->dbg[42] = globaltimer();
    }
    const uint32_t n_prev = ctl->n_prev;
    grid_arrive(&ctl->bar1);
    if (a.warm_params) {
      // the parameter fields the finalize reads, once, so that its phases do not each start with
      // a constant-cache miss (A/B switch AUTX_WARM_PARAMS)
      const unsigned char* pa = reinterpret_cast<const unsigned char*>(&a);
      uint32_t acc = 0;
      for (uint32_t off = tid * 4; off < (uint32_t)offsetof(StepArgs, pro) + 64; off += ST_THREADS * 4)
        acc ^= *reinterpret_cast<const uint32_t*>(pa + off);
      if (acc == 0x9E3779B9u) red32[32] = acc;
    }
    grid_wait(&ctl->bar1, gridDim.x);
    if (stamps && tid == 0) ctl->dbg[43] = globaltimer();
    select_for(a, NONE, S);
    const uint32_t qs = S.qs, mp = S.m, nx = S.nx, n_live = S.n_live, n_promo = S.n_promo;
    finalize_core<I>(a, dsm, qs, mp, nx, n_live, n_promo, n_prev, true, red64, red32);
    return;
  }
  // ---- tile CTA ----
  uint32_t* s_filt = reinterpret_cast<uint32_t*>(dsm);  // 2048-bit filter of completed programs
  const bool filt_on = !a.defer_all && a.pro.n_comp > 0;
  if (filt_on) {
    if (tid < 64) s_filt[tid] = 0;
    __syncthreads();
    if (tid < a.pro.n_comp) {
      const uint32_t p = a.pro.comp_prog[tid];
      atomicOr(&s_filt[(p >> 5) & 63], 1u << (p & 31));
    }
    __syncthreads();
  }
  uint32_t qw[2];
  uint32_t last = NONE;
  if (a.pro_first) {
    if (tid == 0) {
      while (ld_relaxed_u32(&ctl->go_seq) != a.seqno) __nanosleep(20);
      fence_acq_rel();
    }
    __syncthreads();
  }
  for (uint32_t tile = blockIdx.x; tile < a.ntiles; tile += a.n_tile_ctas) {
    uint64_t hq = 0;
    uint32_t np = 0, nl = 0;
    tile_pass(a, tile, s_filt, filt_on, s_filt + 64, qw, hq, np, nl);
    tile_publish(a, tile, hq, np, nl, wq16, wn);
    last = tile;
  }
  grid_arrive(&ctl->bar1);
  if (stamps && tid == 0) atomicMax(&ctl->dbg[48], globaltimer());
  grid_wait(&ctl->bar1, gridDim.x);
  for (uint32_t tile = blockIdx.x; tile < a.ntiles; tile += a.n_tile_ctas) {
    const long long xc0 = clock64();
    select_for(a, tile, S);
    const long long xc1 = clock64();
    if (stamps && tid == 0 && tile == 0) ctl->dbg[54] = globaltimer();
    if (tile != last) {
      // an earlier tile of this CTA: its flags after the pass, from L2
      const uint32_t row0 = tile * TILE + tid * ROWS_PER_THREAD;
      const uint2 qv = row0 < a.n_rows ? __ldcg(reinterpret_cast<const uint2*>(a.ct.qf + row0))
                                       : make_uint2(0x40404040u, 0x40404040u);
      qw[0] = qv.x;
      qw[1] = qv.y;
      last = tile;
    }
    // rows that ran in the previous step: their records go to prev_rec
    const bool run = ((qw[0] | qw[1]) & 0x10101010u) != 0;
    const bool any_run = __syncthreads_or(run);
    if (any_run || S.has) extract_tile(a, tile, qw, S, red64, S.has != 0, dsm + 1024);
    __syncthreads();  // S reuse
    if (stamps && tid == 0) {
      atomicMax(&ctl->dbg[61], (unsigned long long)(xc1 - xc0));            // selection, cycles
      atomicMax(&ctl->dbg[62], (unsigned long long)(clock64() - xc1));      // extraction, cycles
      if (S.has) atomicAdd(&ctl->dbg[63], 1ull);                             // tiles with candidates
      if (any_run) atomicAdd(&ctl->dbg[39], 1ull);                           // tiles with running rows
    }
    if (stamps && tid == 0 && tile == 0) ctl->dbg[55] = globaltimer();
  }
  grid_arrive(&ctl->bar2);
  if (stamps && tid == 0) atomicMax(&ctl->dbg[56], globaltimer());
}

// Radix mode: the finalize alone (one CTA) on the sorted candidates k_take wrote (q* = K: no
// region B; the partition leaves an already key-ordered Y unchanged).
template <int I>
__global__ void __launch_bounds__(ST_THREADS) k_fin(const __grid_constant__ StepArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ unsigned long long red64[33];
  __shared__ uint32_t red32[33];
  Ctl* ctl = a.ctl;
  finalize_core<I>(a, dsm, a.pol.K, 0u, ctl->n_x, ctl->n_live, ctl->n_promoted, ctl->n_prev, false, red64, red32);
}

// ---------------------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------------------
cudaError_t launch_complete(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl,
                            const uint32_t* slots, uint32_t n, uint32_t t, KvState kv, bool kv_on,
                            CompRec* rec_out, bool apply, uint32_t* prev_rec) {
  // size the CTA to the record count: a typical step completes ~BS/mean-decode calls
  if (n <= 32)
    return launch_pdl(k_complete<32>, 1, 32, 0, s, pol, ct, pt, ctl, slots, n, t, kv, kv_on, rec_out, apply, prev_rec);
  else if (n <= 256)
    return launch_pdl(k_complete<256>, 1, 256, 0, s, pol, ct, pt, ctl, slots, n, t, kv, kv_on, rec_out, apply, prev_rec);
  return launch_pdl(k_complete<1024>, 1, 1024, 0, s, pol, ct, pt, ctl, slots, n, t, kv, kv_on, rec_out, apply, prev_rec);
}

cudaError_t launch_apply(cudaStream_t s, const Policy& pol, ProgTable pt, const void* base,
                         uint64_t stride, uint32_t G, uint32_t t) {
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_apply<<<1, 1024, 0, s>>>(pol, pt, (const char*)base, stride, G, t);
  return cudaGetLastError();
}

cudaError_t launch_route(cudaStream_t s, const void* base, uint64_t stride, uint32_t G,
                         const RouteArr* arr, uint32_t n, int8_t* pin, uint32_t threshold,
                         int32_t* out) {
  if (!n) return cudaSuccess;
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_route<<<1, 32, 0, s>>>((const char*)base, stride, G, arr, n, pin, threshold, out);
  return cudaGetLastError();
}

cudaError_t launch_register(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt,
                            const ArrivalRec* recs, uint32_t n, uint32_t first_slot, uint32_t t,
                            const uint32_t* par) {
  if (n == 0) return cudaSuccess;
  return launch_pdl(k_register, (n + 255) / 256, 256, 0, s, pol, ct, pt, recs, n, first_slot, t, par);
}

// Candidates per finalize thread for a batch size (C = ST_THREADS * I >= 2 BS).
static int fin_items(uint32_t bs) { return bs <= 512 ? 2 : bs <= 1024 ? 4 : 8; }

template <int I>
static cudaError_t setup_one(int* occ) {
  const size_t sm = fin_smem_bytes<I>();
  cudaError_t e = cudaFuncSetAttribute(k_step<I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_fin<I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k_step<I>, ST_THREADS, sm);
}

// Called by autx_create with the context's device current (the attributes are per device).
cudaError_t step_kernel_setup(uint32_t max_batch, uint32_t* capacity_out) {
  int dev = 0, sms = 0, occ = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int I = fin_items(max_batch);
  e = I == 2 ? setup_one<2>(&occ) : I == 4 ? setup_one<4>(&occ) : setup_one<8>(&occ);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  *capacity_out = (uint32_t)(occ * sms);
  return cudaSuccess;
}

cudaError_t launch_prologue(cudaStream_t s, const StepArgs& a) {
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_prologue<<<1, ST_THREADS, PRO_INLINE * (4 + sizeof(ArrivalRec) + sizeof(CompRec)), s>>>(a);
  return cudaGetLastError();
}

template <int I>
static cudaError_t launch_step_kernel(cudaStream_t s, const StepArgs& a, uint32_t grid) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ST_THREADS);
  cfg.dynamicSmemBytes = fin_smem_bytes<I>();
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // CTAs wait for each other: all must be resident
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  return cudaLaunchKernelEx(&cfg, k_step<I>, a);
}

template <int I>
static cudaError_t launch_fin_kernel(cudaStream_t s, const StepArgs& a) {
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  k_fin<I><<<1, ST_THREADS, fin_smem_bytes<I>(), s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_step(cudaStream_t s, StepArgs& a, uint32_t capacity, cudaEvent_t* ev, const RadixState* rx,
                        uint32_t arr_base, uint32_t* radix_passes) {
  a.ntiles = std::max<uint32_t>(1, (a.n_rows + TILE - 1) / TILE);
  a.out.n_sup = (a.ntiles + SUP_TILES - 1) / SUP_TILES;
  a.n_tile_ctas = std::min<uint32_t>(a.ntiles, capacity - 1);
  const int I = fin_items(a.pol.max_batch);
  if (ev) cudaEventRecord(ev[0], s);
  cudaError_t e;
  if (rx) {
    if (a.do_pro) {
      e = launch_prologue(s, a);
      if (e != cudaSuccess) return e;
    }
    static int sms = 0;
    if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    e = launch_radix_order(s, a.pol, a.ct, a.pt, a.ctl, a.out, *rx, a.t, a.n_rows, arr_base, sms, radix_passes);
    if (e != cudaSuccess) return e;
    e = I == 2 ? launch_fin_kernel<2>(s, a) : I == 4 ? launch_fin_kernel<4>(s, a) : launch_fin_kernel<8>(s, a);
  } else {
    const uint32_t grid = a.n_tile_ctas + 1;
    e = I == 2 ? launch_step_kernel<2>(s, a, grid) : I == 4 ? launch_step_kernel<4>(s, a, grid)
                                                          : launch_step_kernel<8>(s, a, grid);
  }
  if (e != cudaSuccess) return e;
  if (ev) cudaEventRecord(ev[1], s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// G8: stable compaction of the call table (drop completed rows, keep (arrival, seq) order).
// live[i] = old row of the i-th live row in table order; dst gets rows 0..n_live-1.
// ---------------------------------------------------------------------------------------------
__global__ void k_compact(CallTable src, CallTable dst, const uint32_t* live, uint32_t n_live) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_live) return;
  uint32_t s = live[i];
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

__global__ void k_set_bidx(CallTable ct, const uint32_t* prev_slots, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ct.bidx[prev_slots[i]] = i;
}

cudaError_t launch_set_bidx(cudaStream_t s, CallTable ct, const uint32_t* prev_slots, uint32_t n) {
  if (n == 0) return cudaSuccess;
  ++g_kernel_launches;
  k_set_bidx<<<(n + 255) / 256, 256, 0, s>>>(ct, prev_slots, n);
  return cudaGetLastError();
}

__global__ void k_remap(uint32_t* slots, uint32_t n, const uint32_t* old2new) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) slots[i] = old2new[slots[i]];
}

cudaError_t launch_compact(cudaStream_t s, CallTable src, CallTable dst, const uint32_t* live,
                           uint32_t n_live) {
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  if (n_live) k_compact<<<(n_live + 255) / 256, 256, 0, s>>>(src, dst, live, n_live);
  return cudaGetLastError();
}

cudaError_t launch_remap(cudaStream_t s, uint32_t* slots, uint32_t n, const uint32_t* old2new) {
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  if (n) k_remap<<<(n + 255) / 256, 256, 0, s>>>(slots, n, old2new);
  return cudaGetLastError();
}

}  // namespace autx
