// Internal definitions shared by the autx host code and its sm_100a kernels.
// Nothing here is part of the C ABI (include/autx.h is).
#pragma once
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

namespace autx {

// ---- per-call flag byte (qf) ---------------------------------------------------------------
constexpr uint8_t QF_QMASK = 0x0F;  // queue index q (0 = Q_1, highest priority)
constexpr uint8_t QF_RUN = 0x10;    // in the previous step's batch ("running", key tie R12)
constexpr uint8_t QF_RES = 0x20;    // KV resident on the GPU (eager eviction: == RUN after a step)
constexpr uint8_t QF_DEAD = 0x40;   // empty row (completed call / never used)
constexpr uint8_t QF_DEM = 0x80;    // multi-step (R32): quantum exhausted in a window step, demotion
                                    // pending until the next scheduling point's dense pass

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr int MAX_K = 16;
constexpr int QP_LINES = 16;
constexpr int SUP_TILES = 16;  // tiles per super-tile (the gather's two-level prefix)
constexpr int SCAN_THREADS = 256;
constexpr int ROWS_PER_THREAD = 8;
constexpr int TILE = SCAN_THREADS * ROWS_PER_THREAD;  // rows per scan tile (2048)
constexpr int FIN_THREADS = 1024;
constexpr int MAX_BATCH = 2048;  // BS limit: k_rank keeps 2 BS keys (+ kvb, indices) in shared memory

// Device-resident call table, struct-of-arrays, rows in (arrival, seq) order.  Row index ==
// registration order, so the paper's FCFS tie `seq` is the row index.
struct CallTable {
  uint64_t* cid;     // call id
  uint32_t* prog;    // process-table row of the call's program
  uint32_t* arr;     // arrival step
  uint8_t* qf;       // queue | flags
  uint32_t* base;    // step of the last reset of (wait, mtime): arrival or promotion
  uint32_t* mtime;   // c.model_time since the last reset (Alg. 1 l.25, l.29)
  uint32_t* exec;    // t_k: executed steps, never reset (R6)
  uint32_t* quanta;  // remaining quantum (AUTX_INF = infinite)
  uint32_t* inh;     // service inherited at arrival (Alg. 1 l.11)
  uint32_t* tok;     // input tokens (context)
  uint32_t* loc;     // resident slot (if RES) or host arena page offset (if swapped), else NONE
  uint32_t* hcls;    // host allocation size class (if swapped)
  uint32_t* bidx;    // index in the last batch it joined (valid while QF_RUN: previous-batch index)
};

// Process-table fields the dense pass gathers for every call, packed so that one 16-byte load
// fetches both.
struct __align__(16) PInfo {
  uint32_t svc;               // PLAS: sum of completed t_k; ATLAS: longest critical path (Alg. 1 l.4)
  uint32_t _pad;
  unsigned long long pwait;   // total waiting time of completed calls (W_p)
};

// Process table, one row per program.
struct ProgTable {
  PInfo* info;          // service + waiting time
  uint32_t* last_arr;   // most recent call arrival
  uint32_t* last_comp;  // most recent call completion
  uint32_t* crit;       // AUTX_ATLAS_EQ2: p(c) + t_c of completed calls, by lineage index (Eq. 2)
};

struct Policy {
  int32_t policy;
  uint32_t K;
  uint32_t q_hi[15];
  uint32_t quanta[16];
  uint32_t beta_num, beta_den;
  uint32_t max_batch;      // resident-set capacity BS + X (R32; = BS when X = 0)
  uint32_t run_batch;      // BS: the first run_batch resident calls run
  uint32_t multistep;      // sched_every > 1: demotion deferred to scheduling points (QF_DEM)
  uint32_t kv_budget;
  uint32_t block_tokens;
  uint32_t n_gpu_blocks;
  uint32_t max_blocks_per_call;
  uint32_t host_pages_lo;  // host arena pages (capped to 2^32-1)
  uint32_t bt_shift;       // log2(block_tokens) if a power of two, else 0xFF
  uint32_t stamps;         // record chain stamps (autx_set_timing mode 2)
  int32_t device;          // CUDA device of the context
};

// Step control block in device memory (written by the prologue kernels).
struct Ctl {
  uint32_t t;          // current step
  uint32_t n_rows;     // rows in use (tail)
  uint32_t ntiles;
  uint32_t tiles_done; // last-CTA ticket for the scan kernel
  // selection result (scan kernel's last CTA)
  uint32_t qstar;      // boundary queue (K if all live calls are candidates)
  uint32_t mprime;     // rows of q* to take in table order
  uint32_t n_cand_a;   // candidates from the table scan
  uint32_t n_cand_b;   // extra running candidates of queue q* (previous batch, not in region A)
  uint32_t qs_boundary;  // slot of the m'-th live row of q* (region A's last q* row)
  uint32_t n_promoted;
  uint32_t n_live;
  // finalize results
  uint32_t n_prev;     // previous batch size (slots in prev_slots)
  uint32_t err;        // sticky device error code (autx_status)
  uint32_t err_info;
  uint32_t n_plan_out, n_plan_in;   // swap plan items
  uint32_t swap_serial;             // a swap-in target block was freed by this step's swap-out:
                                    // the directions must run one after the other
  uint32_t plan_out_chunks, plan_in_chunks;
  // allocator state
  uint32_t free_top;       // GPU block free stack size
  uint32_t rs_free_top;    // resident-slot free stack size
  uint32_t host_bump;      // host arena bump pointer (pages)
  uint32_t rank_done;      // last-CTA ticket of k_rank (fused finalize)
  // batch totals reduced by k_rank's list writers (rank_lists), read and reset by finalize
  uint32_t acc_nbatch, acc_nadmit;
  unsigned long long acc_kv, acc_swap_in;
  uint32_t host_free_top[32];  // per size class free-stack size
  // self-selecting gather (default select path): slot + 1 of region A's last q* row (0 = none),
  // and the scan's partial totals, spread over QP_LINES 128-B lines (scan CTA b adds into line
  // b % QP_LINES: same-address reductions serialise at L2): [0, MAX_K) live rows per queue after
  // anti-starvation, [MAX_K] promotions, [MAX_K + 1] live rows.  Reset by finalize.
  uint32_t qs_bnd1;
  uint32_t last_n_b;   // region B size of the last step (autx_step_stats; n_cand_b is reset by finalize)
  // this step's scalars, written by the prologue from its parameters, read by the rest of the
  // chain after its PDL wait: a graph replay then only re-parameterises the prologue node
  uint32_t s_t, s_n_rows, s_seqno, s_n_active;
  uint32_t s_tail_prev;  // rows older than this step's arrivals (finalize / compaction): the scan
                         // may read them before its PDL wait
  uint32_t scan_ticket;  // k_scan_emit: tile ticket (look-back order); reset by finalize
  alignas(128) uint32_t qpart[QP_LINES][32];
  unsigned long long dbg[96];  // [32, 64) live chain stamps, [64, 96) last step's (AUTX_CHAIN_STAMPS)  // %globaltimer stamps of kernel phases (autx_phase_times)
};

// Host-visible step output written by the finalize kernel into mapped pinned memory.
struct HostOut {
  uint32_t n_batch, n_admit, n_preempt, n_active;
  unsigned long long swap_out_blocks, swap_in_blocks, kv_blocks;
  uint32_t n_promoted, err;
  uint32_t seqno;  // step sequence number, for sanity
  uint32_t err_info;
  uint32_t n_standby;  // R32: resident standby calls after the batch in the batch list
  uint32_t _pad;
};
static_assert(sizeof(HostOut) <= 64, "HostOut heads the 64-byte counts block of the output lists");

// Swap plan (built by finalize, executed by autx_kv_swap).
struct PlanItem {
  unsigned long long host_page;  // page offset in the host arena
  uint32_t nblk;                 // number of blocks
  uint32_t blk_off;              // offset into plan block list
};

struct KvState {
  uint32_t* free_stack;     // [n_gpu_blocks]
  uint32_t* rs_free;        // [max_batch] resident-slot free stack
  uint32_t* rs_nblk;        // [max_batch] blocks held per resident slot
  uint32_t* rs_blocks;      // [max_batch * max_blocks_per_call]
  uint32_t* host_free;      // [32][host_free_cap] per-class free stacks of page offsets
  uint32_t host_free_cap;
  PlanItem* plan_out;       // [max_batch]
  PlanItem* plan_in;        // [max_batch]
  uint32_t* plan_out_blocks;   // [kv cap]
  uint32_t* plan_in_blocks;    // [kv cap]
  uint32_t* bt_offsets;     // [max_batch+1] block table CSR of the batch
  uint32_t* bt_blocks;      // [kv cap]
  uint32_t plan_cap;        // capacity of the plan block lists
};

// Candidate record written by the multi-CTA gather so that the single-CTA finalize reads
// contiguous, L2-resident data instead of chasing random rows of the call table.
struct CandRec {
  unsigned long long cid;
  uint32_t slot, arr, tok, exec, mtime, quanta, qf, _pad;
};

#ifdef __CUDACC__
// Unique 64-bit order key (R11, R12): q:4 | arrival relative to step t:27 | not-running:1 |
// seq (row):31.  Requires t - arrival < 2^27 and rows < 2^31.
__device__ __forceinline__ uint64_t cand_key(const CandRec& r, uint32_t t) {
  uint64_t arel = (uint64_t)((1u << 27) - 1 - (t - r.arr)) & ((1u << 27) - 1);  // later arrival: larger
  return ((uint64_t)(r.qf & QF_QMASK) << 59) | (arel << 32) | ((uint64_t)((r.qf & QF_RUN) ? 0u : 1u) << 31) |
         (r.slot & 0x7FFFFFFFu);
}

__device__ __forceinline__ void load_rec(const struct CallTable& ct, uint32_t s, CandRec* r) {
  CandRec x;
  x.cid = ct.cid[s];
  x.slot = s;
  x.arr = ct.arr[s];
  x.tok = ct.tok[s];
  x.exec = ct.exec[s];
  x.mtime = ct.mtime[s];
  x.quanta = ct.quanta[s];
  x.qf = ct.qf[s];
  x._pad = (x.qf & QF_RES) ? ct.bidx[s] : NONE;  // index in the previous resident list
  *r = x;
}
#endif

struct Outputs {
  uint32_t* batch_slots;     // [max_batch]
  uint64_t* batch_ids;       // [max_batch]
  uint64_t* admit_ids;       // [max_batch]
  uint64_t* preempt_ids;     // [max_batch]
  uint32_t* prev_slots;      // [max_batch] previous batch (slots), ctl->n_prev entries
  uint32_t* preempt_slots;   // [max_batch]
  uint32_t* admit_slots;     // [max_batch]
  uint32_t* cand;            // [cand_cap] candidate slots (radix path)
  uint32_t cand_cap;
  CandRec* cand_rec;         // [cand_cap] region-A candidate records
  CandRec* prev_rec;         // [max_batch] records of the previous batch
  uint64_t* ckey;            // [2 BS] keys: region A at [0, nA), previous batch at [nA, nA + n_prev)
  uint64_t* skey;            // [2 BS] keys sorted by k_rank
  uint32_t* sidx;            // [2 BS] element index of each sorted key
  CandRec* srec;             // [2 BS] candidate records in sorted order
  unsigned long long* prev_pos;  // [max_batch] seqno << 32 | sorted position of previous-batch entry j
                                 // (k_rank; entries that are no candidate keep an older seqno)
  uint32_t use_prev_pos;     // finalize tests batch membership of the previous batch by prev_pos
  uint32_t rank_lists;       // k_rank writes batch / admit lists and accounting (no KV allocator)
  uint32_t rank_wide;        // k_rank: a warp per key when the candidates fill <= half its grid
  uint32_t rank_buckets;     // k_rank: O(BS) bucket ranks when region B is empty (else all-pairs count)
  uint32_t prev_early;       // k_finalize: prev_rec was written two kernels back (read before the PDL wait)
  uint32_t* ckvb;            // [2 BS] kvb of each key in ckey (R14)
  uint32_t* tile_cnt;        // [ntiles_cap * MAX_K]
  uint32_t* sup_cnt;         // [ceil(ntiles_cap / SUP_TILES) * MAX_K] per-queue counts of super-tiles
                             // (scan: atomics; gather: prefix; finalize: reset)
  uint32_t* gtile;           // [ntiles_cap] k_gather_ss: 1 if the tile held candidates last step (prefetch hint)
  uint32_t gtile_cap;
  unsigned long long* lb;    // [ntiles_cap * 4] k_scan_emit look-back words (4 queues each; finalize: reset)
  CandRec* cq;               // [MAX_K * max_batch] k_scan_emit: the first max_batch live calls of each
                             // queue, in table order (queue q at q * max_batch)
  HostOut* hout;             // host-visible counts (pinned)
  HostOut* d_hout;           // device copy of the counts (copied out with the lists by one DMA)
  int zero_copy;             // 1: finalize stores the host mirrors itself over PCIe (A/B switch)
  uint64_t* h_batch;         // pinned host mirrors
  uint64_t* h_admit;
  uint64_t* h_preempt;
  uint32_t* h_batch_slots;   // pinned mirror of batch_slots (host-side completion checks)
};

// AUTX_ORDER_RADIX buffers (radix_kernels.cu)
struct RadixState {
  uint64_t* keys;        // [rows padded to 4096]
  uint64_t* keys_alt;
  uint32_t* dig_hist;    // [4][256] global digit histograms (digits 4..7)
  uint32_t* h_dig_hist;  // pinned mirror
  uint32_t* tile_hist;   // [256][ntiles]
};

// Completion record (one per completed call): what UPDATE_PROCESS_TABLE needs.
struct CompRec {
  uint32_t prog;  // process-table row (identical on every rank: rows are created in the
                  // replicated routing order)
  uint32_t exec;  // t_k
  uint32_t cp;    // inh + t_k (ATLAS critical path candidate)
  uint32_t tw;    // total waiting steps
};

// Routing-epoch record of one engine, followed by max_batch CompRec.
struct RouteHdr {
  unsigned long long load;  // queued + running calls after this step's completions (R21)
  uint32_t n_comp;
  uint32_t _pad;
};

struct RouteArr {
  uint32_t prog;
  uint32_t tok;
};

// Arrival record staged by the host.
struct ArrivalRec {
  uint64_t cid;
  uint32_t prog;
  uint32_t tok;
  uint32_t flags;  // bit0: program is new in this batch (inh = 0); bit1: first record of it;
                   // bits 8-31 (AUTX_ATLAS_EQ2): number of DAG parents
  uint32_t par;    // AUTX_ATLAS_EQ2: offset of the parents' lineage indices in PrologueArgs::par
};

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled while its
// predecessor in the stream still runs; it must call pdl_wait() before touching its inputs.
extern unsigned long long g_kernel_launches;  // every library kernel launch (autx_kernel_launches)

// A kernel launch recorded instead of issued (the step's launches are replayed as one CUDA graph
// whose kernel nodes get this step's parameters: see autx_api.cu, step_graph_run).
struct LaunchRec {
  const void* func;
  dim3 grid, block;
  size_t smem;
  std::vector<unsigned char> blob;  // argument values, 16-B aligned each
  std::vector<size_t> off;
  template <typename T>
  void push(const T& v) {
    if (blob.capacity() < 8192) blob.reserve(8192);  // one allocation per record
    const size_t o = (blob.size() + 15) & ~size_t(15);
    blob.resize(o + sizeof(T));
    memcpy(blob.data() + o, &v, sizeof(T));
    off.push_back(o);
  }
  std::vector<void*> ptrs() {
    std::vector<void*> p(off.size());
    for (size_t i = 0; i < off.size(); ++i) p[i] = blob.data() + off[i];
    return p;
  }
};
extern thread_local std::vector<LaunchRec>* g_launch_rec;  // non-null: launch_pdl records into it
extern thread_local size_t g_launch_n;                      // ... at [g_launch_n++] (a pool reused every step)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  if (g_launch_rec) {
    if (g_launch_n == g_launch_rec->size()) g_launch_rec->emplace_back();
    LaunchRec& r = (*g_launch_rec)[g_launch_n++];
    r.blob.clear();
    r.off.clear();
    r.func = reinterpret_cast<const void*>(k);
    r.grid = grid;
    r.block = block;
    r.smem = smem;
    (r.push(static_cast<KArgs>(args)), ...);
    __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);  // runs in the graph replay
    return cudaSuccess;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  __atomic_fetch_add(&g_kernel_launches, 1ull, __ATOMIC_RELAXED);
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Inputs of the fused step prologue (completions + arrivals), passed by value as kernel
// parameters when they fit (PRO_INLINE each), else through the pointers.
#ifndef AUTX_PRO_INLINE
#define AUTX_PRO_INLINE 96
#endif
constexpr int PRO_INLINE = AUTX_PRO_INLINE;
struct PrologueArgs {
  uint32_t n_comp, n_arr, first_slot, t;
  uint32_t n_prog_rows, n_rows, seqno, n_active;  // process-table rows in use; table rows, step seqno, active calls
  const uint32_t* comp_ptr;
  const ArrivalRec* arr_ptr;
  const uint32_t* comp_lin;  // AUTX_ATLAS_EQ2: lineage index of each completion (mapped pinned)
  const uint32_t* par;       // AUTX_ATLAS_EQ2: parents' lineage indices (mapped pinned)
  uint32_t comp[PRO_INLINE];
  uint32_t comp_prog[PRO_INLINE];  // their programs' process-table rows (the host knows them): prefetched
  ArrivalRec arr[PRO_INLINE];
};

// ---- kernel launchers (sched_kernels.cu / swap_kernels.cu) ----------------------------------
cudaError_t launch_complete(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl,
                            const uint32_t* slots, uint32_t n, uint32_t t, KvState kv, bool kv_on,
                            CompRec* rec_out, bool apply);
cudaError_t launch_prologue(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl, KvState kv,
                            bool kv_on, CompRec* rec_out, const PrologueArgs& a);
cudaError_t launch_apply(cudaStream_t s, const Policy& pol, ProgTable pt, const void* base,
                         uint64_t stride, uint32_t G, uint32_t t);
cudaError_t launch_route_hdr(cudaStream_t s, void* rec, uint64_t load, uint32_t n_comp);
cudaError_t launch_route(cudaStream_t s, const void* base, uint64_t stride, uint32_t G,
                         const RouteArr* arr, uint32_t n, int8_t* pin, uint32_t threshold,
                         int32_t* out, uint32_t mode, uint32_t* rr);
cudaError_t launch_register(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt,
                            const ArrivalRec* recs, uint32_t n, uint32_t first_slot, uint32_t t,
                            const uint32_t* par = nullptr);
// Per-device setup of the step kernels (shared-memory attributes); called by autx_create after
// cudaSetDevice.
cudaError_t step_kernels_setup();
cudaError_t launch_step(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl,
                        Outputs out, KvState kv, bool kv_on, uint32_t t, uint32_t n_rows,
                        uint32_t seqno, cudaEvent_t* ev /* 4 events or null */,
                        const RadixState* rx /* non-null: AUTX_ORDER_RADIX */, uint32_t arr_base,
                        uint32_t* radix_passes, bool window = false);
cudaError_t launch_radix_order(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl,
                               Outputs out, RadixState rx, uint32_t t, uint32_t n_rows,
                               uint32_t arr_base, int sms, uint32_t* passes_out);
cudaError_t launch_swap(cudaStream_t s, const Ctl* ctl, KvState kv, void* const* d_kpool,
                        void* const* d_vpool, uint32_t n_layers, uint32_t chunk_bytes,
                        char* host_arena, int direction, int n_ctas);
cudaError_t launch_stage(cudaStream_t s, const Ctl* ctl, KvState kv, void* const* d_kpool,
                         void* const* d_vpool, uint32_t n_layers, uint32_t chunk_bytes,
                         char* staging, int direction, int n_ctas);
cudaError_t launch_compact(cudaStream_t s, CallTable src, CallTable dst, uint32_t n_rows, uint32_t n_live,
                           uint32_t* tile_live, uint32_t* old2new, Ctl* ctl, uint32_t* prev_slots);

}  // namespace autx
