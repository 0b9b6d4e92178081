/*
 * autx.h — C ABI of the B200-native Autellix scheduler hot path (arXiv 2502.13965).
 *
 * One autx_ctx = one serving engine on one GPU ("each LLM engine replica runs in a
 * dedicated process"; here: one process per GPU).  All device work is stream-ordered on the
 * stream given in autx_config.stream.  All arithmetic is integer; time is measured in engine
 * steps (one decode iteration; SURVEY reading R17).  No function throws or aborts: every
 * entry point returns an autx_status and, on failure, leaves a message for autx_last_error().
 * Asynchronous CUDA failures surface as AUTX_E_CUDA from the next call.
 *
 * Citations: P:L<n> = line n of the paper text; "Alg. 1 l.k" = Algorithm 1 line k
 * (P:L149-194); "Alg. 2 l.k" = Algorithm 2 line k; R<n> = reading n of the
 * ambiguity register in DESIGN.md §3 (= SURVEY.md §8(c)).
 *
 * Per-step protocol (SURVEY §8(c) "Oracle step t"; event order of S:L572, reading R10):
 *     autx_complete(ids of calls that finished in step t-1)   -> process-table update  (a1)
 *     autx_register_call(arrivals of step t, canonical order)  -> registration           (a2)
 *     autx_sched_step(t, &out)          demotion, anti-starvation, order, cutoff     (a3-a6)
 *     autx_kv_swap(&layout, &stats)     swap-out of out.preempt, swap-in of out.admit (a7)
 * Multi-engine routing (a8) is autx_route_* (see below).
 */
#ifndef AUTX_H
#define AUTX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct autx_ctx autx_ctx;

typedef enum {
  AUTX_OK = 0,
  AUTX_E_INVAL = 1,  /* bad argument / config, non-canonical arrival order, kvb > P at arrival (R13) */
  AUTX_E_NOENT = 2,  /* unknown call or program id ("missing entry")                      */
  AUTX_E_EXIST = 3,  /* duplicate call id                                                           */
  AUTX_E_NOMEM = 4,  /* call table / program table / GPU block pool / host arena full; kvb > P (R14) */
  AUTX_E_STATE = 5,  /* protocol violation: completing a call that did not run in the last step,
                        registering after sched_step of the same step, step not increasing        */
  AUTX_E_CUDA = 6,   /* CUDA runtime error (possibly from earlier asynchronous work)               */
  AUTX_E_NCCL = 7
} autx_status;

/* AUTX_ATLAS is Alg. 1's scalar ATLAS (every new call inherits its program's longest observed
 * critical path, l.4 / l.11).  AUTX_ATLAS_EQ2 is the exact Eq. 2: a new call
 * inherits max over its parents c_k of p(c_k) + t_k (0 for a root), parents given through
 * autx_register_call_dag; the process table is still updated by Alg. 1 l.4 (it feeds the
 * anti-starvation ratio).  Single-engine only (nranks == 1); reading R31. */
typedef enum { AUTX_FCFS = 0, AUTX_MLFQ = 1, AUTX_PLAS = 2, AUTX_ATLAS = 3, AUTX_ATLAS_EQ2 = 4 } autx_policy;

/* Ordering strategy for step a5 (both produce the identical batch: the key is unique).
 *  AUTX_ORDER_SELECT: top-BS selection over the table kept in (arrival, seq) order.
 *  AUTX_ORDER_RADIX : full stable LSD radix sort, one byte per digit, of packed 64-bit keys
 *                     (queue:4 | arrival:27 | not-running:1 | seq:32) over every active call. */
typedef enum { AUTX_ORDER_SELECT = 0, AUTX_ORDER_RADIX = 1 } autx_order_mode;

#define AUTX_INF 0xFFFFFFFFu /* infinite quantum / budget */

/* Multi-engine routing (a8, f3).  LOCALITY is Alg. 2; the other two are the
 * comparators of §6.4: LEAST_USED sends every call to the engine with the fewest
 * calls in the system (ties -> lowest id, no pinning); ROUND_ROBIN cycles through the engines in
 * canonical arrival order, the cursor persisting across steps (replicated on every rank). */
typedef enum {
  AUTX_ROUTE_LOCALITY = 0,
  AUTX_ROUTE_LEAST_USED = 1,
  AUTX_ROUTE_ROUND_ROBIN = 2
} autx_route_policy;

typedef struct {
  int32_t policy;            /* autx_policy                                                         */
  uint32_t K;                /* number of queues, 1..16                                     */
  uint32_t q_hi[15];         /* PLAS/ATLAS entry bounds Q_i^hi, i < K-1, ascending; queue i covers
                                [q_hi[i-1], q_hi[i]) with q_hi[-1] = 0 and Q_K^hi = inf (R1) */
  uint32_t quanta[16];       /* per-queue quantum in steps, >= 1; AUTX_INF = infinite (Alg. 1 l.13)   */
  uint32_t beta_num;         /* anti-starvation threshold beta = beta_num / beta_den    */
  uint32_t beta_den;         /* 0 -> beta = infinity: never promote (R3)                             */
  uint32_t max_batch;        /* BS, 1..4096 (P:L184 can_fit)                                          */
  uint32_t kv_budget_blocks; /* P: KV blocks the batch may hold; AUTX_INF = unbounded (R13, R14)     */
  uint32_t block_tokens;     /* tokens per KV block (16); kvb(c) = ceil((input+exec+1)/block_tokens) */
  uint32_t max_calls;        /* call-table rows (active calls + completed holes before compaction)   */
  uint32_t max_programs;     /* process-table rows                                                   */
  uint32_t token_threshold;  /* Alg. 2 l.2 short/long threshold (2048)                               */
  uint32_t order_mode;       /* autx_order_mode                                                      */
  uint32_t n_gpu_blocks;     /* GPU KV pool size in blocks; 0 disables the block allocator/swap      */
  uint32_t max_blocks_per_call; /* block-table width per resident call                              */
  uint64_t host_pages;       /* host swap arena size in logical blocks (pages)                       */
  int32_t device;            /* CUDA device ordinal                                                  */
  void* stream;              /* cudaStream_t all device work is ordered on (e.g.
                                torch.cuda.current_stream().cuda_stream); NULL = the legacy default
                                stream                                                               */
  int32_t rank, nranks;      /* engine id and engine count (routing)                                 */
  uint32_t route_policy;     /* autx_route_policy: how autx_route places arrivals        */
  uint32_t _reserved;        /* must be 0                                                            */
  void* nccl_comm;           /* ncclComm_t of the nranks engines (autx_comm_init), caller-owned, or
                                NULL: autx_route then needs nranks == 1 (the split
                                autx_route_pack/apply path needs no communicator)                     */
  /* Multi-step scheduling with over-provisioning ("running the scheduler once every N
   * decoding steps ... overprovisions queued requests already on the GPU"; reading R32):     */
  uint32_t sched_every;      /* N >= 1 (0 = 1): the ordering runs at the first step, every N-th step
                                after the last one and whenever the carried resident list is empty;
                                the steps between (window steps) keep the resident list, in order,
                                under the KV budget.  N > 1: single engine, AUTX_ORDER_SELECT      */
  uint32_t overprovision;    /* X >= 0: the resident set is the longest prefix with <= BS + X calls
                                (BS + X <= 2048); its first BS calls run, the rest are standby    */
} autx_config;

/* One arriving LLM call (Alg. 1 l.9).  Arrays of these must be in canonical order
 * (arrival_step, program_arrival_step, program_id, call_id); arrival_step must equal
 * the step of the next autx_sched_step.  input_tokens = full input context (drives kvb and
 * Alg. 2's LEN, R21). */
typedef struct {
  uint64_t call_id;
  uint64_t program_id;
  uint32_t arrival_step;
  uint32_t program_arrival_step;
  uint32_t input_tokens;
  uint32_t _pad;
} autx_call_desc;

/* Result of one scheduling step.  Device lists stay valid until the next autx_sched_step;
 * the host mirrors (pinned, library-owned) and the counts are valid once `done` (a
 * cudaEvent_t) has completed — autx_step_wait() waits for it. */
typedef struct {
  const uint64_t* batch;       /* device: call ids of the batch, in key order (Alg. 1 l.32-39),
                                  then the standby calls (n_standby, R32)                      */
  const uint64_t* admit;       /* device: batch (and standby) calls not resident before this step,
                                  batch order                                                    */
  const uint64_t* preempt;     /* device: resident calls no longer resident, previous order; a
                                  preempted call that never ran has no KV content to swap (R32)  */
  const uint64_t* h_batch;     /* host mirrors of the three lists                                */
  const uint64_t* h_admit;
  const uint64_t* h_preempt;
  uint32_t n_batch, n_admit, n_preempt, n_active;
  uint64_t swap_out_blocks;    /* sum over preempt of held blocks ceil((input+exec)/bt)  (R15) */
  uint64_t swap_in_blocks;     /* sum over admit with a host copy of held blocks               */
  uint64_t kv_blocks;          /* sum over the batch of kvb                                    */
  uint32_t n_promoted;         /* anti-starvation promotions this step (diagnostic)            */
  uint32_t n_standby;          /* R32: resident standby calls; batch[n_batch .. n_batch+n_standby)
                                  (device and host lists) holds them in order; 0 when X = 0      */
  void* done;                  /* cudaEvent_t recorded after the step's device work            */
} autx_step_out;

/* Caller-owned paged KV pools (vLLM-style): for layer l, k_pool[l] and
 * v_pool[l] are device base pointers of [n_gpu_blocks][chunk_bytes] arrays; one (layer, K|V,
 * block) chunk is chunk_bytes.  host_arena: pinned (cudaHostAlloc / torch pin_memory) buffer
 * of host_pages * n_layers * 2 * chunk_bytes bytes; a swapped call occupies one contiguous
 * range laid out [block][layer][K|V][chunk] ("consolidate all KV blocks into a single
 * contiguous chunk").  Pointer arrays are host arrays read during the call. */
typedef struct {
  void* const* k_pool;
  void* const* v_pool;
  uint32_t n_layers;
  uint32_t chunk_bytes;       /* multiple of 16 */
  void* host_arena;
  uint64_t host_arena_bytes;
} autx_kv_layout;

typedef enum { AUTX_SWAP_SM = 0, AUTX_SWAP_PER_CHUNK_MEMCPY = 1, AUTX_SWAP_STAGED_DMA = 2 } autx_swap_mode;

typedef struct {
  uint64_t bytes_d2h, bytes_h2d;  /* bytes moved over the host link by this call               */
  uint32_t chunks_d2h, chunks_h2d;
  float ms;                       /* device time of the swap (CUDA events), valid after return */
  uint32_t duplex;                /* 1: swap-out and swap-in ran at the same time (full duplex)  */
} autx_swap_stats;

/* ---- lifecycle -------------------------------------------------------------------------- */
autx_status autx_create(const autx_config* cfg, autx_ctx** out);
autx_status autx_destroy(autx_ctx* ctx);
const char* autx_last_error(const autx_ctx* ctx);   /* never NULL; "" when no error */
const char* autx_version(void);

/* ---- per-step calls (host arrays, borrowed for the duration of the call) ------------------ */
/* start_session: optional explicit program creation; register_call creates on first
 * sight.  E_EXIST if the program exists. */
autx_status autx_start_program(autx_ctx* ctx, uint64_t program_id);
/* end_session: removes the process-table entry.  E_STATE if the program still
 * has active calls; E_NOENT if unknown. */
autx_status autx_end_program(autx_ctx* ctx, uint64_t program_id);
/* Calls that finished decoding in the previous step (Alg. 1 l.16-18, UPDATE_PROCESS_TABLE
 * l.1-7).  Each must have been in the previous batch (E_STATE) and be known (E_NOENT). Blocks
 * until the previous step's `done`. */
autx_status autx_complete(autx_ctx* ctx, const uint64_t* call_ids, uint32_t n);
/* Arrivals of the current step (Alg. 1 l.9-14), canonical order (E_INVAL otherwise).  Under
 * AUTX_ATLAS_EQ2 these are roots (Eq. 2: priority 0). */
autx_status autx_register_call(autx_ctx* ctx, const autx_call_desc* calls, uint32_t n);
/* AUTX_ATLAS_EQ2 arrivals with their DAG parents ("its parents P(c_j) in the same
 * program"; the DAG is learned as calls arrive).  parent_offsets: host array of n+1
 * ascending offsets into parent_ids (host array of call ids); call i's parents are
 * parent_ids[parent_offsets[i] .. parent_offsets[i+1]).  Every parent must be a call of the
 * same program that has completed (autx_complete, this step or earlier) and whose program has
 * not ended: unknown id -> E_NOENT, still active -> E_STATE, other program -> E_INVAL.  The
 * priority p(c_i) = max_k p(c_k) + t_k is computed on the device from the parents' completion
 * records (a call with no parents is a root: 0).  Other policies: E_INVAL.  The completed
 * calls' p + t values are kept until their program ends (capacity 4 x max_calls: E_NOMEM). */
autx_status autx_register_call_dag(autx_ctx* ctx, const autx_call_desc* calls, uint32_t n,
                                   const uint32_t* parent_offsets, const uint64_t* parent_ids);
/* One scheduling step t (Alg. 1 l.15-39): demotion, anti-starvation, ordering, cutoff,
 * admit/preempt lists, step accounting.  t must increase by >= 1 per call (steps with no
 * active call may be skipped). */
autx_status autx_sched_step(autx_ctx* ctx, uint32_t step, autx_step_out* out);
autx_status autx_step_wait(autx_ctx* ctx, autx_step_out* out);  /* waits for out->done, fills counts */
/* One whole engine step in one call (Alg. 1 l.1-39 for step t): exactly autx_complete(completed,
 * n_completed) if n_completed > 0, then autx_end_program for each of ended_programs[n_ended],
 * then autx_register_call(arrivals, n_arrivals) if n_arrivals > 0, then autx_sched_step(t) and
 * autx_step_wait — the same operations, arguments and errors as those calls, in that order,
 * stopping at the first error.  All arrays are host memory owned by the caller (may be NULL
 * when their count is 0).  For the serving loop that has nothing to overlap with the step:
 * one boundary crossing instead of five.  Not for AUTX_ATLAS_EQ2 arrivals with parents (use
 * autx_register_call_dag) or multi-engine contexts (autx_route must run between them: E_STATE). */
autx_status autx_step(autx_ctx* ctx, uint32_t step, const uint64_t* completed, uint32_t n_completed,
                      const uint64_t* ended_programs, uint32_t n_ended, const autx_call_desc* arrivals,
                      uint32_t n_arrivals, autx_step_out* out);

/* ---- KV swap (a7) --------------------------------------------------------------------- */
/* Executes the last step's swap plan: swap-out (GPU blocks -> host arena) of every preempted
 * call and swap-in (host arena -> newly allocated GPU blocks) of every admitted call with a
 * host copy.  The two directions run at the same time (full duplex: both halves of the host
 * link; SM mode one kernel, staged-DMA mode a second stream) unless a swap-in target block was
 * freed by this step's swap-out — the allocator hands out blocks freed in earlier steps first,
 * so that only happens when the pool runs short — then swap-out runs first.  Requires
 * n_gpu_blocks > 0. */
autx_status autx_kv_swap(autx_ctx* ctx, const autx_kv_layout* layout, int32_t mode,
                         autx_swap_stats* stats);
/* Block table of the last batch as CSR: d_offsets[n_batch+1], d_blocks[...] (device pointers,
 * valid until the next autx_sched_step). */
autx_status autx_block_table(autx_ctx* ctx, const uint32_t** d_offsets, const uint32_t** d_blocks);
/* Host copy of the same CSR: h_offsets[n_batch+1] (capacity max_batch+1), h_blocks[cap]. */
autx_status autx_block_table_host(autx_ctx* ctx, uint32_t* h_offsets, uint32_t* h_blocks, uint32_t cap,
                                  uint32_t* n_batch);

/* ---- multi-engine routing (a8, Alg. 2) --------------------------------------------------- */
/* One routing epoch as ONE collective call (Alg. 2 "query engine workloads in
 * parallel"; SURVEY §8(e) order).  Every rank calls it once per step, after autx_complete and
 * before autx_register_call, with the identical replicated arrival batch `calls` (canonical
 * order, host array, n may be 0).  On the ctx stream it
 *   1. writes this engine's epoch record: load = queued + running calls after this step's
 *      completions (R21) and the completion records of autx_complete (device resident),
 *   2. all-gathers the nranks fixed-size records with ncclAllGather on cfg.nccl_comm (NVLink /
 *      NVSwitch; with nranks == 1 and no communicator the record is used in place),
 *   3. applies all nranks engines' completion records (its own included) to the replicated
 *      process table (sums / maxima commute, so every rank's table stays identical, R22),
 *   4. routes `calls` with the policy of cfg.route_policy (Alg. 2: LEN <= token_threshold ->
 *      least-loaded engine, else the program's pinned engine, pinning on first sight; loads from
 *      the epoch snapshot, incremented per assignment, R23); pins are replicated.
 * engine_out[i] (host array, n entries) receives the engine of calls[i]; it is the call's only
 * host round trip (the caller registers the calls routed to it).  Errors: E_INVAL (nranks > 1
 * without nccl_comm, non-canonical batch, > 8 engines), E_STATE (after autx_register_call, or
 * twice in one step), E_NCCL (the collective failed; message from ncclGetErrorString). */
autx_status autx_route(autx_ctx* ctx, const autx_call_desc* calls, uint32_t n, int32_t* engine_out);

/* NCCL communicator helpers for autx_config.nccl_comm (the library links NCCL itself; torch is
 * only the launcher).  Rank 0 calls autx_comm_unique_id (128 bytes), the caller broadcasts the
 * bytes to every rank (any channel), then every rank calls autx_comm_init with its own rank and
 * device (collective).  The communicator outlives every ctx that uses it: destroy it last. */
autx_status autx_comm_unique_id(void* id_out /* 128 bytes */);
autx_status autx_comm_init(const void* id /* 128 bytes */, int32_t rank, int32_t nranks, int32_t device,
                           void** comm_out);
autx_status autx_comm_destroy(void* comm);

/* Routing epoch, split around the caller's own all-gather (e.g. gloo on a host): pack this
 * engine's epoch record (load = queued + running calls after this step's completions, R21, and
 * the completion records of this step) into a device buffer of autx_route_record_bytes(), then
 * after the all-gather of nranks records apply the peers' completion records to the
 * replicated process table (R22) and route `calls` (replicated, canonical order) with Alg. 2;
 * engine_out[i] receives the engine of calls[i] (host array); pins are replicated. */
uint64_t autx_route_record_bytes(const autx_ctx* ctx);
autx_status autx_route_pack(autx_ctx* ctx, void* d_record);
autx_status autx_route_apply(autx_ctx* ctx, const void* d_records, const autx_call_desc* calls,
                             uint32_t n, int32_t* engine_out);

/* ---- introspection for tests and benchmarks -------------------------------------------- */
typedef struct {
  uint64_t call_id;
  uint32_t q, quanta, wait, mtime, exec, totwait, inh, input_tokens, arrival_step, flags;
} autx_call_state;                 /* flags: 1 running, 2 resident, 4 host copy */
/* Copies the state of every active call, in (arrival, seq) order, as of the end of the last
 * sched_step, to a host array of capacity `cap`; *n receives the count. */
autx_status autx_dump_calls(autx_ctx* ctx, autx_call_state* out, uint32_t cap, uint32_t* n);
autx_status autx_program_state(autx_ctx* ctx, uint64_t program_id, uint32_t* svc, uint64_t* pwait);
/* Shape of the last step's selection (select mode; radix mode reports q* = K, region B = 0):
 * q* = the smallest queue with sum_{k<=q*} live_k >= BS (K if none), m' = rows of q* taken in
 * table order, region A = the rows below q* plus those m' rows, region B = running calls of q*
 * past them in the same arrival group, the table rows scanned, the live
 * programs and the live calls per queue after anti-starvation.  Synchronises the stream. */
typedef struct {
  uint32_t qstar, mprime, n_x, n_b;
  uint32_t n_rows, n_programs;
  uint32_t queue_counts[16];
} autx_selection_stats;
autx_status autx_step_stats(autx_ctx* ctx, autx_selection_stats* out);
/* Device-time of the kernels of the last sched_step (CUDA events around each phase). */
typedef struct { float complete_ms, register_ms, scan_ms, select_ms, finalize_ms, total_ms; } autx_step_timing;
autx_status autx_last_step_timing(autx_ctx* ctx, autx_step_timing* t);
autx_status autx_set_timing(autx_ctx* ctx, int32_t on);
uint32_t autx_num_active(const autx_ctx* ctx);
/* %globaltimer stamps (ns) recorded inside the kernels of the last step, for profiling:
 * [0..8] k_finalize phases, [16..19] k_complete phases, and in a -DAUTX_CHAIN_STAMPS build
 * [64 + 3k, 64 + 3k + 2] = (CTA 0 past griddepcontrol.wait, latest CTA end, latest CTA past the
 * wait) of chain kernel k (0 prologue, 1 scan, 2 select, 3 gather, 4 rank, 5 finalize; 0 = did
 * not run), [84, 85] = (ranked keys, key slots) of k_rank; copies min(cap, 96). */
autx_status autx_phase_times(autx_ctx* ctx, uint64_t* ns, uint32_t cap);
/* G8 stable compactions of the call table so far (device kernels into the other half of a double
 * buffer; run inside autx_register_call when the table's tail reaches max_calls) and the host time
 * they took (id-map remap), in microseconds. */
autx_status autx_compaction_stats(const autx_ctx* ctx, uint64_t* n_compactions, double* host_us);
/* Number of kernels this library has launched so far (all contexts of the process). */
uint64_t autx_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* AUTX_H */
