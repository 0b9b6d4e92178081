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
constexpr uint8_t QF_INB = 0x80;    // scratch: member of the batch being formed (finalize only)

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr int MAX_K = 16;
constexpr int QP_LINES = 16;
constexpr int SUP_TILES = 16;  // tiles per super-tile (the two-level queue-count prefix)
constexpr int ST_THREADS = 512;  // threads per CTA of the step kernel
constexpr int ROWS_PER_THREAD = 8;
constexpr int TILE = ST_THREADS * ROWS_PER_THREAD;  // rows per tile (4096)
constexpr int MAX_BATCH = 2048;  // BS limit: the finalize keeps 2 BS candidate records in shared memory

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
  uint32_t max_batch;
  uint32_t kv_budget;
  uint32_t block_tokens;
  uint32_t n_gpu_blocks;
  uint32_t max_blocks_per_call;
  uint32_t host_pages_lo;  // host arena pages (capped to 2^32-1)
  uint32_t bt_shift;       // log2(block_tokens) if a power of two, else 0xFF
  uint32_t stamps;         // record chain stamps (autx_set_timing mode 2)
};

// Step control block in device memory.
struct Ctl {
  uint32_t t;          // current step
  uint32_t n_x;        // candidates of region A (radix path: set by k_take)
  uint32_t qstar;      // boundary queue q* of the last step (K: every live call is a candidate)
  uint32_t mprime;     // rows of q* taken in table order
  uint32_t n_promoted, n_live;  // radix path: reduced by k_keys (the step kernel uses qpart)
  uint32_t n_prev;     // previous batch size (slots in prev_slots)
  uint32_t err;        // sticky device error code (autx_status)
  uint32_t err_info;
  uint32_t n_plan_out, n_plan_in;   // swap plan items
  uint32_t plan_out_chunks, plan_in_chunks;
  // allocator state
  uint32_t free_top;       // GPU block free stack size
  uint32_t rs_free_top;    // resident-slot free stack size
  uint32_t host_bump;      // host arena bump pointer (pages)
  uint32_t bnd_slot, bnd_arr;  // region A's last row of q* (slot, arrival): published by its tile
  uint32_t n_b;                // region B size of the last step (finalize; autx_step_stats)
  uint32_t host_free_top[32];  // per size class free-stack size
  // step-kernel synchronisation, one 128-B line each: the prologue's completion (step seqno) and
  // the two grid barriers (arrival counts, reset by the finalize CTA at the end of the step)
  alignas(128) uint32_t pro_seq;
  alignas(128) uint32_t go_seq;   // AUTX_PRO_FIRST: the prologue's loads are issued (tiles may stream)
  alignas(128) uint32_t bar1;
  alignas(128) uint32_t bar2;
  // scan partial totals over QP_LINES 128-B lines (CTA b adds into line b % QP_LINES: same-address
  // reductions serialise at L2): [MAX_K] promotions, [MAX_K + 1] live rows.  Reset by finalize.
  alignas(128) uint32_t qpart[QP_LINES][32];
  unsigned long long dbg[96];  // %globaltimer stamps (autx_phase_times): [40, 56) this step, [64, 80) last step
};

// Host-visible step output written by the finalize kernel into mapped pinned memory.
struct HostOut {
  uint32_t n_batch, n_admit, n_preempt, n_active;
  unsigned long long swap_out_blocks, swap_in_blocks, kv_blocks;
  uint32_t n_promoted, err;
  uint32_t seqno;  // step sequence number, for sanity
  uint32_t err_info;
};

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

// Candidate records, struct-of-arrays: a row among the step's <= BS smallest keys (region A) at
// its position in (queue, seq) order, or a row of the previous batch at its previous-batch index.
// Written by the tile CTAs with coalesced stores, read by the finalize with coalesced loads.
struct RecSoA {
  unsigned long long* cid;
  uint32_t* slot;
  uint32_t* arr;
  uint32_t* tok;
  uint32_t* exec;
  uint32_t* mt;    // mtime after this step's anti-starvation
  uint32_t* qt;    // quanta after this step's anti-starvation
  uint32_t* qfb;   // qf | previous-batch index << 8 (valid while QF_RUN); QF_DEAD: completed
};

struct Outputs {
  uint32_t* batch_slots;     // [max_batch]
  uint64_t* batch_ids;       // [max_batch]
  uint64_t* admit_ids;       // [max_batch]
  uint64_t* preempt_ids;     // [max_batch]
  uint32_t* prev_slots;      // [max_batch] previous batch (slots), ctl->n_prev entries
  uint32_t* preempt_slots;   // [max_batch]
  uint32_t* admit_slots;     // [max_batch]
  RecSoA xs;                 // [max_batch] region A in (queue, seq) order
  RecSoA ps;                 // [max_batch] the previous batch's rows by previous-batch index: written by
                             // the tiles owning them (live rows, after the dense pass) and by the
                             // prologue (completed rows: qfb = QF_DEAD)
  uint32_t* tile_cnt;        // [ntiles_cap * MAX_K] live rows per (tile, queue) after anti-starvation
  uint32_t* sup_cnt;         // [ceil(ntiles_cap / SUP_TILES) * MAX_K] per-queue counts of super-tiles
                             // (scan: atomics; selection: prefix; finalize: reset)
  uint32_t n_sup;            // super-tiles in use this step (set per launch; finalize resets them)
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

extern unsigned long long g_kernel_launches;  // every library kernel launch (autx_kernel_launches)

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled while its
// predecessor in the stream still runs; it must call pdl_wait() before touching its inputs.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
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

// Inputs of the step prologue (completions + arrivals), passed by value as kernel parameters
// when they fit (PRO_INLINE each), else through the pointers.  comp_prog[i] is the process-table
// row of completion i (a host-side id map, no arithmetic): the scan CTAs defer exactly the rows
// of those programs until the prologue has updated their service.
constexpr int PRO_INLINE = 128;
struct PrologueArgs {
  uint32_t n_comp, n_arr, first_slot, t;
  uint32_t n_prog_rows, _pad[3];  // process-table rows in use
  const uint32_t* comp_ptr;
  const ArrivalRec* arr_ptr;
  const uint32_t* comp_lin;  // AUTX_ATLAS_EQ2: lineage index of each completion (mapped pinned)
  const uint32_t* par;       // AUTX_ATLAS_EQ2: parents' lineage indices (mapped pinned)
  uint32_t comp[PRO_INLINE];
  uint32_t comp_prog[PRO_INLINE];
  ArrivalRec arr[PRO_INLINE];
};

// Everything one scheduling step reads, passed to the step kernel as one __grid_constant__
// parameter block.
struct StepArgs {
  Policy pol;
  CallTable ct;
  ProgTable pt;
  Ctl* ctl;
  Outputs out;
  KvState kv;
  CompRec* rec_out;     // this step's completion records (routing epoch)
  uint32_t kv_on;
  uint32_t t, n_rows, ntiles;
  uint32_t n_tile_ctas;  // CTAs 0 .. n_tile_ctas-1 scan tiles; CTA n_tile_ctas runs prologue + finalize
  uint32_t seqno;
  uint32_t first_new;   // first row registered by this step's prologue (rows below are older)
  uint32_t defer_all;   // the prologue's records are not inline: every row waits for it
  uint32_t do_pro;      // the step has a prologue (completions or arrivals)
  uint32_t pro_first;   // the tiles start streaming only once the prologue's loads are issued
  uint32_t warm_params; // the finalize CTA touches its parameter fields while it waits
  PrologueArgs pro;
};

// ---- kernel launchers (sched_kernels.cu / swap_kernels.cu / radix_kernels.cu) ---------------
cudaError_t launch_complete(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl,
                            const uint32_t* slots, uint32_t n, uint32_t t, KvState kv, bool kv_on,
                            CompRec* rec_out, bool apply, uint32_t* prev_qfb);
// The step prologue (a1, a2) as its own kernel (radix mode, bulk bursts, before a compaction).
cudaError_t launch_prologue(cudaStream_t s, const StepArgs& a);
cudaError_t launch_apply(cudaStream_t s, const Policy& pol, ProgTable pt, const void* base,
                         uint64_t stride, uint32_t G, uint32_t t);
cudaError_t launch_route(cudaStream_t s, const void* base, uint64_t stride, uint32_t G,
                         const RouteArr* arr, uint32_t n, int8_t* pin, uint32_t threshold,
                         int32_t* out);
cudaError_t launch_register(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt,
                            const ArrivalRec* recs, uint32_t n, uint32_t first_slot, uint32_t t,
                            const uint32_t* par = nullptr);
cudaError_t launch_set_bidx(cudaStream_t s, CallTable ct, const uint32_t* prev_slots, uint32_t n);
// Per-device launch setup of the step kernels (shared-memory attribute, co-resident CTA
// capacity); called by autx_create after cudaSetDevice.
cudaError_t step_kernel_setup(uint32_t max_batch, uint32_t* capacity_out);
// One scheduling step (a1-a6): the cooperative step kernel (select mode), or the prologue, the
// radix sort and the finalize kernel (radix mode).  ev: 2 events around the step, or null.
cudaError_t launch_step(cudaStream_t s, StepArgs& a, uint32_t capacity, cudaEvent_t* ev,
                        const RadixState* rx, uint32_t arr_base, uint32_t* radix_passes);
cudaError_t launch_radix_order(cudaStream_t s, const Policy& pol, CallTable ct, ProgTable pt, Ctl* ctl,
                               Outputs out, RadixState rx, uint32_t t, uint32_t n_rows,
                               uint32_t arr_base, int sms, uint32_t* passes_out);
cudaError_t launch_swap(cudaStream_t s, const Ctl* ctl, KvState kv, void* const* d_kpool,
                        void* const* d_vpool, uint32_t n_layers, uint32_t chunk_bytes,
                        char* host_arena, int direction, int n_ctas);
cudaError_t launch_stage(cudaStream_t s, const Ctl* ctl, KvState kv, void* const* d_kpool,
                         void* const* d_vpool, uint32_t n_layers, uint32_t chunk_bytes,
                         char* staging, int direction, int n_ctas);
cudaError_t launch_compact(cudaStream_t s, CallTable src, CallTable dst, const uint32_t* live,
                           uint32_t n_live);
cudaError_t launch_remap(cudaStream_t s, uint32_t* slots, uint32_t n, const uint32_t* old2new);

}  // namespace autx
