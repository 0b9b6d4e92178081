// Host side of the autx C ABI (include/autx.h): context, id maps, protocol checks, staging.
// All scheduling arithmetic runs in the sm_100a kernels (sched_kernels.cu, swap_kernels.cu);
// this file only validates, maps 64-bit ids to table rows, stages records in pinned memory
// and launches.
#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include <nccl.h>

#include "../../include/autx.h"
#include "autx_internal.cuh"
#include "idmap.h"

using namespace autx;

unsigned long long autx::g_kernel_launches = 0;
thread_local std::vector<autx::LaunchRec>* autx::g_launch_rec = nullptr;
thread_local size_t autx::g_launch_n = 0;

extern "C" uint64_t autx_kernel_launches(void) {
  return __atomic_load_n(&g_kernel_launches, __ATOMIC_RELAXED);
}

struct autx_ctx {
  autx_config cfg{};
  Policy pol{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  CallTable ct{};
  CallTable ct2{};                 // the other half of the double-buffered call table (compaction)
  size_t rows = 0;                 // call-table rows (max_calls padded to whole tiles)
  uint32_t* d_tile_live = nullptr; // compaction: live rows per tile
  uint32_t* d_old2new = nullptr;   // compaction: old row -> new row (NONE: dropped)
  std::vector<uint32_t> h_old2new;
  uint64_t n_compactions = 0;
  double compact_host_us = 0;
  ProgTable pt{};
  Ctl* ctl = nullptr;
  Outputs out{};
  KvState kv{};
  bool kv_on = false;
  // pinned staging (device reads it through UVA)
  uint32_t* h_cslots = nullptr;  // [max_batch * 4] completion slots
  std::vector<uint32_t> cprog;    // process-table row of each staged completion (prologue prefetch hint)
  std::vector<autx::LaunchRec> rec_pool;  // the step's recorded launches (graph replay), reused
  uint32_t cslots_cap = 0;
  ArrivalRec* h_arr = nullptr;
  uint32_t arr_cap = 0;
  uint32_t* d_cslots = nullptr;
  ArrivalRec* d_arr = nullptr;
  // host-side maps
  IdMap call_slot;                                    // active call id -> row
  IdMap prog_row;                                     // program id -> process-table row
  std::vector<uint32_t> prog_free;
  uint32_t prog_next = 0;
  std::vector<uint32_t> prog_active;                  // active calls per program row
  std::vector<uint32_t> slot_prog;                    // row -> program row (host mirror)
  std::vector<uint32_t> slot_arr;                     // row -> arrival step (host mirror)
  std::vector<uint8_t> slot_live;                     // row -> active?
  uint32_t low = 0;                                   // no live row below this one
  RadixState rx{};
  bool radix = false;
  uint32_t radix_passes = 0;
  // slots of the last step's batch: ran_seq[slot] == seqno (from the mirrored batch slots)
  std::vector<uint32_t> ran_seq;
  bool last_batch_valid = false;
  std::vector<uint32_t> comp_scratch;
  uint32_t tail = 0;
  // protocol state
  bool stepped = false;       // at least one sched_step done
  uint32_t t_last = 0;        // last step scheduled
  bool pending_done = false;  // a sched_step whose `done` was not waited on
  uint32_t pend_t = 0;        // step the pending records belong to (0 = unset)
  bool pend_set = false;
  bool completed_this = false, registered_this = false;
  uint32_t n_completed_pending = 0;
  uint64_t last_key[4] = {0, 0, 0, 0};
  bool have_last_key = false;
  uint32_t seqno = 0;
  cudaEvent_t done = nullptr;
  bool timing = false;
  cudaEvent_t ev[8] = {};
  autx_step_timing last_timing{};
  // kv swap scratch
  void** d_pools = nullptr;  // [2 * n_layers]
  uint32_t pools_cap = 0;
  void** h_pools = nullptr;
  char* staging = nullptr;          // swap-out staging (staged DMA mode)
  size_t staging_bytes = 0;
  char* staging_in = nullptr;       // swap-in staging: its own buffer, so the legs overlap
  size_t staging_in_bytes = 0;
  cudaStream_t stream_in = nullptr; // the swap-in leg's stream (full duplex, staged DMA mode)
  cudaEvent_t sev_in[2] = {};
  bool last_swap_duplex = false;
  cudaEvent_t sev[2] = {};
  char* d_outblk = nullptr;  // [counts | batch | admit | preempt] on the device
  char* h_outblk = nullptr;  // pinned mirror
  size_t outblk_bytes = 0;
  // routing epoch (a8)
  char* d_route_local = nullptr;   // RouteHdr + max_batch CompRec: this step's completion records
  char* d_route_all = nullptr;     // nranks gathered records (autx_route's all-gather destination)
  int8_t* d_pin = nullptr;         // [max_programs] Alg. 2 pin table (-1 = none)
  uint32_t* d_rr = nullptr;        // Round Robin cursor (replicated: every rank routes the same batch)
  RouteArr* h_rarr = nullptr;
  RouteArr* d_rarr = nullptr;
  int32_t* d_rout = nullptr;
  uint32_t rarr_cap = 0;
  bool routed_this = false;
  // R32 multi-step scheduling: steps since the last scheduling point (0: none yet)
  uint32_t since = 0;
  uint32_t n_reg_this = 0;
  // work staged for the next sched_step's prologue kernel (single-engine mode)
  uint32_t n_comp_staged = 0, n_arr_staged = 0, arr_first_slot = 0;
  std::unordered_set<uint64_t> staged_new_progs;
  // AUTX_ATLAS_EQ2 (Eq. 2): every call of a live program holds a lineage index; at
  // completion the device stores p(c) + t_c there, and arrivals name their parents' indices
  bool eq2 = false;
  std::unordered_map<uint64_t, uint32_t> lin_of;   // call id -> lineage index
  std::vector<uint32_t> lin_prog;                  // lineage index -> program row
  std::vector<std::vector<uint64_t>> prog_calls;   // program row -> its calls' ids (lineage holders)
  std::vector<uint32_t> lin_free;
  uint32_t lin_next = 0, lin_cap = 0;
  uint32_t* h_clin = nullptr;                      // [cslots_cap] lineage of each completion (pinned)
  uint32_t* h_par = nullptr;                       // parents' lineage indices of staged arrivals (pinned)
  uint32_t par_cap = 0, n_par_staged = 0;
  // the step's kernels replayed as a CUDA graph: one executable per launch signature (kernels,
  // block shapes, shared memory), whose kernel nodes receive each step's parameters
  struct StepGraph {
    std::vector<const void*> funcs;
    std::vector<dim3> blocks;
    std::vector<size_t> smem;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t x = nullptr;
    std::vector<cudaGraphNode_t> nodes;
    std::vector<std::vector<unsigned char>> blobs;  // parameters last set on each node
    std::vector<dim3> grids;
  };
  std::vector<StepGraph> graphs;
  cudaStream_t cap_stream = nullptr;  // capture only (the legacy stream cannot be captured)
  bool timed_complete = false, timed_register = false;   // events 4-5 / 6-7 recorded this step
  bool tc_step = false, tr_step = false;                  // ... for the step being waited on
  std::string err;
};

// AUTX_HOST_PROFILE=1: host time per section of autx_sched_step, printed by autx_destroy.
struct HostProf {
  const bool on = getenv("AUTX_HOST_PROFILE") != nullptr;
  double acc[8] = {};
  uint64_t n = 0;
  std::chrono::steady_clock::time_point t0;
  void start() { if (on) t0 = std::chrono::steady_clock::now(); }
  void lap(int i) {
    if (!on) return;
    const auto t1 = std::chrono::steady_clock::now();
    acc[i] += std::chrono::duration<double, std::micro>(t1 - t0).count();
    t0 = t1;
  }
};
static HostProf g_hp;

static autx_status fail(autx_ctx* c, autx_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(ctx, AUTX_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                            \
  } while (0)

template <typename T>
static cudaError_t dalloc(T** p, size_t n) {
  return cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
}

extern "C" const char* autx_version(void) { return "autx 0.1 (sm_100a)"; }

extern "C" const char* autx_last_error(const autx_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

static autx_status alloc_tables(autx_ctx* ctx) {
  const autx_config& c = ctx->cfg;
  size_t rows = ((size_t)c.max_calls + TILE - 1) / TILE * TILE;  // padded to whole tiles
  ctx->rows = rows;
  for (CallTable* tp : {&ctx->ct, &ctx->ct2}) {  // double buffer: compaction writes the other one
    CallTable& t = *tp;
    CK(dalloc(&t.cid, rows)); CK(dalloc(&t.prog, rows)); CK(dalloc(&t.arr, rows));
    CK(dalloc(&t.qf, rows)); CK(dalloc(&t.base, rows)); CK(dalloc(&t.mtime, rows));
    CK(dalloc(&t.exec, rows)); CK(dalloc(&t.quanta, rows)); CK(dalloc(&t.inh, rows));
    CK(dalloc(&t.tok, rows)); CK(dalloc(&t.loc, rows)); CK(dalloc(&t.hcls, rows)); CK(dalloc(&t.bidx, rows));
    CK(cudaMemsetAsync(t.qf, QF_DEAD, rows, ctx->stream));
    CK(cudaMemsetAsync(t.prog, 0, rows * 4, ctx->stream));
    CK(cudaMemsetAsync(t.base, 0, rows * 4, ctx->stream));
    CK(cudaMemsetAsync(t.mtime, 0, rows * 4, ctx->stream));
  }
  CK(dalloc(&ctx->d_tile_live, rows / TILE + 1));
  CK(dalloc(&ctx->d_old2new, rows));
  ProgTable& p = ctx->pt;
  size_t P = std::max<uint32_t>(c.max_programs, 1);
  CK(dalloc(&p.info, P)); CK(dalloc(&p.last_arr, P)); CK(dalloc(&p.last_comp, P));
  CK(cudaMemsetAsync(p.info, 0, P * sizeof(PInfo), ctx->stream));
  CK(dalloc(&ctx->ctl, 1));
  CK(cudaMemsetAsync(ctx->ctl, 0, sizeof(Ctl), ctx->stream));
  Outputs& o = ctx->out;
  uint32_t BS = ctx->pol.max_batch;  // list / resident-set capacity: BS + X (R32)
  size_t ntiles = rows / TILE + 1;
  // one device block [counts | batch | admit | preempt | batch slots] and its pinned mirror: one
  // D2H per step (the slots let the host check completions without an id set)
  const uint32_t BSp = (BS + 1) & ~1u;  // even list strides keep every list 16-byte aligned
  const uint32_t BS4 = (BS + 3) & ~3u;
  ctx->outblk_bytes = 64 + (size_t)3 * BSp * 8 + (size_t)BS4 * 4;
  CK(cudaMalloc((void**)&ctx->d_outblk, ctx->outblk_bytes));
  CK(cudaHostAlloc((void**)&ctx->h_outblk, ctx->outblk_bytes, cudaHostAllocMapped));
  memset(ctx->h_outblk, 0, ctx->outblk_bytes);
  // zero-copy mirrors from finalize (default) vs one D2H DMA after it: measured equal-or-better
  o.zero_copy = getenv("AUTX_DMA_OUT") == nullptr;
  o.d_hout = reinterpret_cast<HostOut*>(ctx->d_outblk);
  o.batch_ids = reinterpret_cast<uint64_t*>(ctx->d_outblk + 64);
  o.admit_ids = o.batch_ids + BSp;
  o.preempt_ids = o.admit_ids + BSp; CK(dalloc(&o.prev_slots, BS)); CK(dalloc(&o.preempt_slots, BS));
  o.batch_slots = reinterpret_cast<uint32_t*>(o.preempt_ids + BSp);
  CK(dalloc(&o.admit_slots, BS));
  o.cand_cap = 2 * BS;
  CK(dalloc(&o.cand, o.cand_cap));
  CK(dalloc(&o.cand_rec, o.cand_cap));
  CK(dalloc(&o.prev_rec, BS));
  CK(dalloc(&o.ckey, 2 * BS));
  CK(dalloc(&o.ckvb, 2 * BS));
  CK(dalloc(&o.skey, 2 * BS));
  CK(dalloc(&o.sidx, 2 * BS));
  CK(dalloc(&o.srec, 2 * BS));
  CK(dalloc(&o.prev_pos, BS));
  CK(cudaMemsetAsync(o.prev_pos, 0, (size_t)BS * 8, ctx->stream));  // seqno 0 never matches
  CK(dalloc(&o.tile_cnt, ntiles * MAX_K));
  CK(dalloc(&o.sup_cnt, (ntiles / SUP_TILES + 1) * MAX_K));
  CK(cudaMemsetAsync(o.sup_cnt, 0, (ntiles / SUP_TILES + 1) * MAX_K * sizeof(uint32_t), ctx->stream));
  CK(dalloc(&o.gtile, ntiles));
  o.gtile_cap = (uint32_t)ntiles;
  CK(cudaMemsetAsync(o.gtile, 0, ntiles * sizeof(uint32_t), ctx->stream));
  CK(dalloc(&o.lb, ntiles * 4));
  CK(cudaMemsetAsync(o.lb, 0, ntiles * 4 * sizeof(unsigned long long), ctx->stream));
  CK(dalloc(&o.cq, (size_t)MAX_K * BS));
  o.hout = reinterpret_cast<HostOut*>(ctx->h_outblk);
  o.h_batch = reinterpret_cast<uint64_t*>(ctx->h_outblk + 64);
  o.h_admit = o.h_batch + BSp;
  o.h_preempt = o.h_admit + BSp;
  o.h_batch_slots = reinterpret_cast<uint32_t*>(o.h_preempt + BSp);
  ctx->ran_seq.assign(rows, 0);
  ctx->cslots_cap = 4 * BS;
  ctx->cprog.assign(PRO_INLINE, 0);
  CK(cudaHostAlloc((void**)&ctx->h_cslots, ctx->cslots_cap * 4, cudaHostAllocMapped));
  ctx->arr_cap = 4 * BS;
  CK(cudaHostAlloc((void**)&ctx->h_arr, ctx->arr_cap * sizeof(ArrivalRec), cudaHostAllocMapped));
  CK(dalloc(&ctx->d_cslots, ctx->cslots_cap));
  CK(dalloc(&ctx->d_arr, ctx->arr_cap));
  CK(dalloc(&ctx->d_route_local, sizeof(RouteHdr) + (size_t)BS * sizeof(CompRec)));
  CK(cudaMemsetAsync(ctx->d_route_local, 0, sizeof(RouteHdr), ctx->stream));
  CK(dalloc(&ctx->d_route_all, (size_t)std::max(c.nranks, 1) * (sizeof(RouteHdr) + (size_t)BS * sizeof(CompRec))));
  CK(dalloc(&ctx->d_pin, P));
  CK(cudaMemsetAsync(ctx->d_pin, 0xff, P, ctx->stream));
  CK(dalloc(&ctx->d_rr, 1));
  CK(cudaMemsetAsync(ctx->d_rr, 0, 4, ctx->stream));
  ctx->prog_active.assign(P, 0);
  ctx->slot_prog.assign(rows, 0);
  ctx->slot_arr.assign(rows, 0);
  ctx->slot_live.assign(rows, 0);
  if (c.policy == AUTX_ATLAS_EQ2) {
    ctx->eq2 = true;
    ctx->lin_cap = (uint32_t)std::min<uint64_t>(4ull * c.max_calls, 0xFFFFFFF0ull);
    CK(dalloc(&p.crit, ctx->lin_cap));
    ctx->lin_prog.assign(ctx->lin_cap, 0);
    ctx->prog_calls.assign(P, {});
    CK(cudaHostAlloc((void**)&ctx->h_clin, ctx->cslots_cap * 4, cudaHostAllocMapped));
    ctx->par_cap = 16 * BS;
    CK(cudaHostAlloc((void**)&ctx->h_par, (size_t)ctx->par_cap * 4, cudaHostAllocMapped));
  }
  if (c.order_mode == AUTX_ORDER_RADIX) {
    ctx->radix = true;
    size_t npad = (rows + 4095) / 4096 * 4096;
    CK(dalloc(&ctx->rx.keys, npad));
    CK(dalloc(&ctx->rx.keys_alt, npad));
    CK(dalloc(&ctx->rx.dig_hist, 4 * 256));
    CK(cudaHostAlloc((void**)&ctx->rx.h_dig_hist, 4 * 256 * 4, 0));
    CK(dalloc(&ctx->rx.tile_hist, 256 * (npad / 4096)));
  }
  // KV block allocator
  if (c.n_gpu_blocks > 0) {
    CK(cudaStreamSynchronize(ctx->stream));  // the async memsets above precede the copies below
    ctx->kv_on = true;
    KvState& kv = ctx->kv;
    uint32_t W = c.max_blocks_per_call;
    CK(dalloc(&kv.free_stack, c.n_gpu_blocks));
    CK(dalloc(&kv.rs_free, BS)); CK(dalloc(&kv.rs_nblk, BS));
    CK(dalloc(&kv.rs_blocks, (size_t)BS * W));
    CK(cudaMemsetAsync(kv.rs_nblk, 0, BS * 4, ctx->stream));
    // free stacks: block ids n-1..0 so that pops hand out 0,1,2,... first
    std::vector<uint32_t> fs(c.n_gpu_blocks), rs(BS);
    for (uint32_t i = 0; i < c.n_gpu_blocks; ++i) fs[i] = c.n_gpu_blocks - 1 - i;
    for (uint32_t i = 0; i < BS; ++i) rs[i] = BS - 1 - i;
    CK(cudaMemcpyAsync(kv.free_stack, fs.data(), fs.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(kv.rs_free, rs.data(), rs.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    uint64_t hp = std::min<uint64_t>(c.host_pages, 0xFFFFFFF0ull);
    kv.host_free_cap = (uint32_t)std::max<uint64_t>(hp, 1);
    CK(dalloc(&kv.host_free, (size_t)32 * kv.host_free_cap));
    CK(dalloc(&kv.plan_out, BS)); CK(dalloc(&kv.plan_in, BS));
    kv.plan_cap = c.n_gpu_blocks;
    CK(dalloc(&kv.plan_out_blocks, kv.plan_cap)); CK(dalloc(&kv.plan_in_blocks, kv.plan_cap));
    CK(dalloc(&kv.bt_offsets, BS + 1)); CK(dalloc(&kv.bt_blocks, kv.plan_cap));
    Ctl init{};
    memset(&init, 0, sizeof init);
    init.free_top = c.n_gpu_blocks;
    init.rs_free_top = BS;
    CK(cudaMemcpyAsync(ctx->ctl, &init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));  // fs, rs, init go out of scope
  }
  return AUTX_OK;
}

extern "C" autx_status autx_create(const autx_config* cfg, autx_ctx** outp) {
  if (!cfg || !outp) return AUTX_E_INVAL;
  *outp = nullptr;
  autx_ctx* ctx = new autx_ctx();
  const autx_config& c = *cfg;
  auto bad = [&](const char* m) {
    autx_status s = fail(ctx, AUTX_E_INVAL, "config: %s", m);
    fprintf(stderr, "autx_create: %s\n", ctx->err.c_str());
    delete ctx;
    return s;
  };
  if (c.policy < AUTX_FCFS || c.policy > AUTX_ATLAS_EQ2) return bad("policy");
  if (c.policy == AUTX_ATLAS_EQ2 && c.nranks > 1) return bad("AUTX_ATLAS_EQ2 is single-engine (nranks must be 1)");
  if (c.route_policy > AUTX_ROUTE_ROUND_ROBIN) return bad("route_policy");
  if (c._reserved) return bad("_reserved must be 0");
  if (c.nranks < 1 || c.nranks > 8 || c.rank < 0 || c.rank >= c.nranks) return bad("rank / nranks (1..8 engines)");
  if (c.K < 1 || c.K > 16) return bad("K must be 1..16");
  for (uint32_t i = 0; i + 1 < c.K; ++i) {
    if (i > 0 && c.q_hi[i] < c.q_hi[i - 1]) return bad("q_hi must be ascending");
  }
  for (uint32_t i = 0; i < c.K; ++i)
    if (c.quanta[i] == 0) return bad("quanta must be >= 1");
  if (c.max_batch < 1 || c.max_batch > (uint32_t)MAX_BATCH) return bad("max_batch must be 1..2048");
  if (c.block_tokens < 1) return bad("block_tokens");
  if (c.max_calls < 1 || c.max_programs < 1) return bad("capacities");
  if (c.max_calls > 0x7FFFFFFFu) return bad("max_calls too large");
  if (c.n_gpu_blocks > 0 && (c.max_blocks_per_call < 1 || c.host_pages < 1))
    return bad("n_gpu_blocks needs max_blocks_per_call and host_pages");
  if (c.n_gpu_blocks > 0 && c.kv_budget_blocks != AUTX_INF && c.kv_budget_blocks > c.n_gpu_blocks)
    return bad("kv_budget_blocks exceeds n_gpu_blocks");
  if (c.order_mode != AUTX_ORDER_SELECT && c.order_mode != AUTX_ORDER_RADIX) return bad("order_mode");
  const uint32_t N = c.sched_every ? c.sched_every : 1u;
  if (c.overprovision > (uint32_t)MAX_BATCH || c.max_batch + c.overprovision > (uint32_t)MAX_BATCH)
    return bad("max_batch + overprovision must be <= 2048");
  if ((N > 1 || c.overprovision) && (c.order_mode != AUTX_ORDER_SELECT || c.nranks > 1))
    return bad("multi-step scheduling / over-provisioning (R32) needs AUTX_ORDER_SELECT and one engine");
  ctx->cfg = c;
  Policy& p = ctx->pol;
  p.policy = c.policy;
  p.K = c.K;
  memcpy(p.q_hi, c.q_hi, sizeof p.q_hi);
  memcpy(p.quanta, c.quanta, sizeof p.quanta);
  p.beta_num = c.beta_num;
  p.beta_den = c.beta_den;
  p.max_batch = c.max_batch + c.overprovision;  // resident set: BS + X (R32)
  p.run_batch = c.max_batch;
  p.multistep = N > 1 ? 1u : 0u;
  p.kv_budget = c.kv_budget_blocks;
  p.block_tokens = c.block_tokens;
  p.bt_shift = 0xFFu;
  if ((c.block_tokens & (c.block_tokens - 1)) == 0)
    for (uint32_t b = 0; b < 32; ++b)
      if ((1u << b) == c.block_tokens) p.bt_shift = b;
  p.n_gpu_blocks = c.n_gpu_blocks;
  p.max_blocks_per_call = c.max_blocks_per_call;
  p.host_pages_lo = (uint32_t)std::min<uint64_t>(c.host_pages, 0xFFFFFFF0ull);
  ctx->device = c.device;
  p.device = c.device;
  if (cudaSetDevice(c.device) != cudaSuccess) {
    autx_status s = fail(ctx, AUTX_E_CUDA, "cudaSetDevice(%d) failed", c.device);
    delete ctx;
    return s;
  }
  if (cudaError_t e = step_kernels_setup(); e != cudaSuccess) {
    autx_status s = fail(ctx, AUTX_E_CUDA, "step kernel setup: %s", cudaGetErrorString(e));
    fprintf(stderr, "autx_create: %s\n", ctx->err.c_str());
    delete ctx;
    return s;
  }
  // NULL = the legacy default stream (what torch.cuda.current_stream() is by default), so
  // library work orders with the caller's default-stream work
  ctx->stream = (cudaStream_t)c.stream;
  ctx->call_slot.reserve(c.max_calls);
  ctx->prog_row.reserve(c.max_programs);
  autx_status s = alloc_tables(ctx);
  if (s == AUTX_OK) {
    if (cudaEventCreateWithFlags(&ctx->done, cudaEventDisableTiming) != cudaSuccess) s = AUTX_E_CUDA;
    for (auto& e : ctx->ev) cudaEventCreate(&e);
    for (auto& e : ctx->sev) cudaEventCreate(&e);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) s = fail(ctx, AUTX_E_CUDA, "init sync");
  }
  if (s != AUTX_OK) {
    fprintf(stderr, "autx_create: %s\n", ctx->err.c_str());
    autx_destroy(ctx);
    return s;
  }
  *outp = ctx;
  return AUTX_OK;
}

extern "C" autx_status autx_destroy(autx_ctx* ctx) {
  if (!ctx) return AUTX_E_INVAL;
  if (g_hp.on && g_hp.n)
    fprintf(stderr, "autx host us/step over %llu sched_steps: checks %.2f prologue %.2f record %.2f graph %.2f tail %.2f\n",
            (unsigned long long)g_hp.n, g_hp.acc[0] / g_hp.n, g_hp.acc[1] / g_hp.n, g_hp.acc[2] / g_hp.n,
            g_hp.acc[3] / g_hp.n, g_hp.acc[4] / g_hp.n);
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (CallTable* tp : {&ctx->ct, &ctx->ct2}) {
    CallTable& t = *tp;
    void* cols[] = {t.cid, t.prog, t.arr, t.qf, t.base, t.mtime, t.exec, t.quanta, t.inh, t.tok, t.loc, t.hcls, t.bidx};
    for (void* p : cols) if (p) cudaFree(p);
  }
  void* dev[] = {ctx->d_tile_live, ctx->d_old2new, ctx->out.prev_pos, ctx->pt.info, ctx->pt.last_arr, ctx->pt.last_comp, ctx->pt.crit,
                 ctx->ctl, ctx->d_outblk, ctx->out.prev_slots, ctx->out.preempt_slots,
                 ctx->out.admit_slots, ctx->out.cand, ctx->out.cand_rec, ctx->out.prev_rec, ctx->out.ckey, ctx->out.ckvb, ctx->out.skey, ctx->out.sidx, ctx->out.srec, ctx->out.tile_cnt, ctx->out.sup_cnt, ctx->out.lb, ctx->out.cq, ctx->out.gtile, ctx->d_cslots, ctx->d_arr, ctx->kv.free_stack, ctx->kv.rs_free,
                 ctx->kv.rs_nblk, ctx->kv.rs_blocks, ctx->kv.host_free, ctx->kv.plan_out,
                 ctx->kv.plan_in, ctx->kv.plan_out_blocks, ctx->kv.plan_in_blocks,
                 ctx->kv.bt_offsets, ctx->kv.bt_blocks, ctx->d_pools, ctx->staging,
                 ctx->d_route_local, ctx->d_route_all, ctx->d_pin, ctx->d_rr, ctx->d_rarr, ctx->d_rout,
                 ctx->rx.keys, ctx->rx.keys_alt, ctx->rx.dig_hist, ctx->rx.tile_hist};
  for (void* p : dev) if (p) cudaFree(p);
  void* host[] = {ctx->h_outblk,
                  ctx->h_cslots, ctx->h_arr, ctx->h_pools, ctx->h_rarr, ctx->h_clin, ctx->h_par,
                  ctx->rx.h_dig_hist};
  for (void* p : host) if (p) cudaFreeHost(p);
  for (auto& g : ctx->graphs) {
    if (g.x) cudaGraphExecDestroy(g.x);
    if (g.g) cudaGraphDestroy(g.g);
  }
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->done) cudaEventDestroy(ctx->done);
  for (auto& e : ctx->ev) if (e) cudaEventDestroy(e);
  for (auto& e : ctx->sev) if (e) cudaEventDestroy(e);
  for (auto& e : ctx->sev_in) if (e) cudaEventDestroy(e);
  if (ctx->stream_in) cudaStreamDestroy(ctx->stream_in);
  if (ctx->staging_in) cudaFree(ctx->staging_in);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return AUTX_OK;
}

// Wait for the last step and make its batch available to the host-side protocol checks.
static autx_status sync_last(autx_ctx* ctx) {
  if (ctx->pending_done) {
    CK(cudaEventSynchronize(ctx->done));
    ctx->pending_done = false;
  }
  if (!ctx->last_batch_valid) {
    if (ctx->stepped) {
      const HostOut& h = *ctx->out.hout;
      if (h.err)
        return fail(ctx, (autx_status)h.err, "device error %u (site %u: 1 host arena full, 2 call needs more "
                    "than max_blocks_per_call, 3 no resident slot, 4 GPU block pool empty, other: head call "
                    "needs more than P) in step %u", h.err, h.err_info, ctx->t_last);
      const uint32_t* bs = ctx->out.h_batch_slots;
      for (uint32_t i = 0; i < h.n_batch; ++i) ctx->ran_seq[bs[i]] = ctx->seqno;
    }
    ctx->last_batch_valid = true;
  }
  return AUTX_OK;
}

static uint32_t next_step(const autx_ctx* ctx) { return ctx->stepped ? ctx->t_last + 1 : 0; }

// Creates a process-table entry (session start): zeroed service/wait, no pin.
static autx_status new_program(autx_ctx* ctx, uint64_t pid, uint32_t* row_out) {
  uint32_t row;
  if (!ctx->prog_free.empty()) { row = ctx->prog_free.back(); ctx->prog_free.pop_back(); }
  else if (ctx->prog_next < ctx->cfg.max_programs) row = ctx->prog_next++;
  else return fail(ctx, AUTX_E_NOMEM, "process table full (%u programs)", ctx->cfg.max_programs);
  ctx->prog_row[pid] = row;
  ctx->prog_active[row] = 0;
  // zero the entry (stream-ordered before any later kernel reads it)
  CK(cudaMemsetAsync(ctx->pt.info + row, 0, sizeof(PInfo), ctx->stream));
  CK(cudaMemsetAsync(ctx->d_pin + row, 0xff, 1, ctx->stream));
  if (row_out) *row_out = row;
  return AUTX_OK;
}

extern "C" autx_status autx_start_program(autx_ctx* ctx, uint64_t pid) {
  if (!ctx) return AUTX_E_INVAL;
  if (ctx->prog_row.count(pid)) return fail(ctx, AUTX_E_EXIST, "program %llu exists", (unsigned long long)pid);
  return new_program(ctx, pid, nullptr);
}

extern "C" autx_status autx_end_program(autx_ctx* ctx, uint64_t pid) {
  if (!ctx) return AUTX_E_INVAL;
  uint32_t* it = ctx->prog_row.find(pid);
  if (!it) return fail(ctx, AUTX_E_NOENT, "unknown program %llu", (unsigned long long)pid);
  if (ctx->prog_active[*it] != 0)
    return fail(ctx, AUTX_E_STATE, "program %llu still has %u active calls", (unsigned long long)pid,
                ctx->prog_active[*it]);
  if (ctx->eq2) {  // the program's Eq. 2 operands go with it
    for (uint64_t cid : ctx->prog_calls[*it]) {
      auto l = ctx->lin_of.find(cid);
      ctx->lin_free.push_back(l->second);
      ctx->lin_of.erase(l);
    }
    ctx->prog_calls[*it].clear();
  }
  ctx->prog_free.push_back(*it);
  ctx->prog_row.erase(pid);
  return AUTX_OK;
}

extern "C" autx_status autx_complete(autx_ctx* ctx, const uint64_t* ids, uint32_t n) {
  if (!ctx || (n && !ids)) return AUTX_E_INVAL;
  if (n == 0) return AUTX_OK;
  autx_status s = sync_last(ctx);
  if (s) return s;
  if (ctx->registered_this)
    return fail(ctx, AUTX_E_STATE, "autx_complete after autx_register_call in the same step");
  if (ctx->completed_this)
    return fail(ctx, AUTX_E_STATE, "autx_complete called twice in one step");
  if (n > ctx->cfg.max_batch) return fail(ctx, AUTX_E_INVAL, "too many completions (%u)", n);
  if (ctx->routed_this) return fail(ctx, AUTX_E_STATE, "autx_complete after autx_route_apply");
  // validate everything before mutating anything
  std::vector<uint32_t>& sl = ctx->comp_scratch;
  sl.resize(n);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t* it = ctx->call_slot.find(ids[i]);
    if (!it) return fail(ctx, AUTX_E_NOENT, "unknown call %llu", (unsigned long long)ids[i]);
    if (!ctx->stepped || ctx->ran_seq[*it] != ctx->seqno)
      return fail(ctx, AUTX_E_STATE, "call %llu did not run in step %u", (unsigned long long)ids[i], ctx->t_last);
    sl[i] = *it;
  }
  {
    std::vector<uint32_t> srt(sl);
    std::sort(srt.begin(), srt.end());
    if (std::adjacent_find(srt.begin(), srt.end()) != srt.end()) return fail(ctx, AUTX_E_INVAL, "duplicate completion");
  }
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t slot = sl[i];
    ctx->h_cslots[i] = slot;
    if (i < (uint32_t)PRO_INLINE) ctx->cprog[i] = ctx->slot_prog[slot];
    if (ctx->eq2) ctx->h_clin[i] = ctx->lin_of.at(ids[i]);
    ctx->slot_live[slot] = 0;
    ctx->prog_active[ctx->slot_prog[slot]] -= 1;
    ctx->call_slot.erase(ids[i]);
    ctx->ran_seq[slot] = 0;
  }
  uint32_t t = next_step(ctx);
  if (ctx->cfg.nranks <= 1) {
    ctx->n_comp_staged = n;  // applied by the next sched_step's prologue kernel
  } else {
    // multi-engine: the records are needed now by autx_route_pack
    if (ctx->timing) cudaEventRecord(ctx->ev[4], ctx->stream);
    CompRec* recs = reinterpret_cast<CompRec*>(ctx->d_route_local + sizeof(RouteHdr));
    CK(launch_complete(ctx->stream, ctx->pol, ctx->ct, ctx->pt, ctx->ctl, ctx->h_cslots, n, t, ctx->kv,
                       ctx->kv_on, recs, false));
    if (ctx->timing) {
      cudaEventRecord(ctx->ev[5], ctx->stream);
      ctx->timed_complete = true;
    }
  }
  ctx->completed_this = true;
  ctx->n_completed_pending = n;
  return AUTX_OK;
}

static autx_status compact(autx_ctx* ctx);

// Launches the staged completions and arrivals of step t: one prologue kernel whose inputs ride
// in the kernel parameters when small; bulk arrivals (an offline burst) go through one DMA and
// the multi-CTA registration kernel.
// always: launch the prologue even without records (sched_step: it also hands the step's scalars
// to the rest of the chain).
static autx_status flush_staged(autx_ctx* ctx, uint32_t t, bool always = false) {
  if (ctx->n_comp_staged == 0 && ctx->n_arr_staged == 0 && !always) return AUTX_OK;
  const bool bulk = ctx->n_arr_staged > 4096;
  PrologueArgs a;
  memset(&a, 0, offsetof(PrologueArgs, comp));
  a.n_comp = ctx->n_comp_staged;
  a.n_arr = bulk ? 0 : ctx->n_arr_staged;
  a.first_slot = ctx->arr_first_slot;
  a.t = t;
  a.n_prog_rows = ctx->prog_next;
  a.n_rows = ctx->tail;
  a.seqno = ctx->seqno;
  a.n_active = (uint32_t)ctx->call_slot.size();
  // larger batches: one DMA each to device memory ahead of the step (stream-ordered before the
  // prologue; the pinned staging is not reused before this step's `done`), read by the kernel from
  // HBM instead of one PCIe round trip per record
  if (a.n_comp <= (uint32_t)PRO_INLINE) {
    memcpy(a.comp, ctx->h_cslots, a.n_comp * sizeof(uint32_t));
    memcpy(a.comp_prog, ctx->cprog.data(), a.n_comp * sizeof(uint32_t));
  } else {
    CK(cudaMemcpyAsync(ctx->d_cslots, ctx->h_cslots, (size_t)a.n_comp * 4, cudaMemcpyHostToDevice, ctx->stream));
    a.comp_ptr = ctx->d_cslots;
  }
  if (a.n_arr <= (uint32_t)PRO_INLINE) {
    memcpy(a.arr, ctx->h_arr, a.n_arr * sizeof(ArrivalRec));
  } else {
    CK(cudaMemcpyAsync(ctx->d_arr, ctx->h_arr, (size_t)a.n_arr * sizeof(ArrivalRec), cudaMemcpyHostToDevice,
                       ctx->stream));
    a.arr_ptr = ctx->d_arr;
  }
  a.comp_lin = ctx->h_clin;  // AUTX_ATLAS_EQ2 only (read through UVA)
  a.par = ctx->h_par;
  CompRec* recs = reinterpret_cast<CompRec*>(ctx->d_route_local + sizeof(RouteHdr));
  if (ctx->timing) cudaEventRecord(ctx->ev[4], ctx->stream);
  CK(launch_prologue(ctx->stream, ctx->pol, ctx->ct, ctx->pt, ctx->ctl, ctx->kv, ctx->kv_on, recs, a));
  if (ctx->timing) {
    cudaEventRecord(ctx->ev[5], ctx->stream);
    ctx->timed_complete = true;
  }
  if (bulk) {
    if (ctx->timing) cudaEventRecord(ctx->ev[6], ctx->stream);
    CK(cudaMemcpyAsync(ctx->d_arr, ctx->h_arr, (size_t)ctx->n_arr_staged * sizeof(ArrivalRec),
                       cudaMemcpyHostToDevice, ctx->stream));
    CK(launch_register(ctx->stream, ctx->pol, ctx->ct, ctx->pt, ctx->d_arr, ctx->n_arr_staged,
                       ctx->arr_first_slot, t, ctx->h_par));
    if (ctx->timing) {
      cudaEventRecord(ctx->ev[7], ctx->stream);
      ctx->timed_register = true;
    }
  }
  ctx->n_comp_staged = ctx->n_arr_staged = 0;
  ctx->n_par_staged = 0;
  // (clear() on an unordered_set memsets every bucket: after a burst of new programs that is
  // ~30k buckets per step, so an empty set is left alone and a big one is released)
  if (ctx->staged_new_progs.size() > 4096) std::unordered_set<uint64_t>().swap(ctx->staged_new_progs);
  else if (!ctx->staged_new_progs.empty()) ctx->staged_new_progs.clear();
  return AUTX_OK;
}

static autx_status register_impl(autx_ctx* ctx, const autx_call_desc* calls, uint32_t n, const uint32_t* poff,
                                 const uint64_t* pids);

extern "C" autx_status autx_register_call(autx_ctx* ctx, const autx_call_desc* calls, uint32_t n) {
  return register_impl(ctx, calls, n, nullptr, nullptr);
}

extern "C" autx_status autx_register_call_dag(autx_ctx* ctx, const autx_call_desc* calls, uint32_t n,
                                              const uint32_t* poff, const uint64_t* pids) {
  if (!ctx) return AUTX_E_INVAL;
  if (!ctx->eq2) return fail(ctx, AUTX_E_INVAL, "autx_register_call_dag needs policy AUTX_ATLAS_EQ2");
  if (n && !poff) return AUTX_E_INVAL;
  return register_impl(ctx, calls, n, poff, pids);
}

static autx_status register_impl(autx_ctx* ctx, const autx_call_desc* calls, uint32_t n, const uint32_t* poff,
                                 const uint64_t* pids) {
  if (!ctx || (n && !calls)) return AUTX_E_INVAL;
  if (n == 0) return AUTX_OK;
  autx_status s = sync_last(ctx);
  if (s) return s;
  const uint32_t t = calls[0].arrival_step;
  if (t < next_step(ctx)) return fail(ctx, AUTX_E_INVAL, "arrival_step %u is in the past", t);
  if (!ctx->call_slot.empty() && t != next_step(ctx))
    return fail(ctx, AUTX_E_STATE, "steps may only be skipped when no call is active");
  if (ctx->completed_this && t != next_step(ctx))
    return fail(ctx, AUTX_E_STATE, "arrivals after completions must be for step %u", next_step(ctx));
  if (ctx->pend_set && ctx->pend_t != t) return fail(ctx, AUTX_E_INVAL, "arrivals of two steps in one batch");
  // validate: canonical order, uniqueness, capacities, kvb <= P (R13)
  std::unordered_map<uint64_t, int> new_prog_seen;
  uint32_t new_progs = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const autx_call_desc& d = calls[i];
    if (d.arrival_step != t) return fail(ctx, AUTX_E_INVAL, "mixed arrival steps in one batch");
    uint64_t key[4] = {d.arrival_step, d.program_arrival_step, d.program_id, d.call_id};
    const uint64_t* prev = ctx->have_last_key ? ctx->last_key : nullptr;
    if (i > 0) {
      const autx_call_desc& q = calls[i - 1];
      uint64_t pk[4] = {q.arrival_step, q.program_arrival_step, q.program_id, q.call_id};
      prev = nullptr;
      if (!std::lexicographical_compare(pk, pk + 4, key, key + 4))
        return fail(ctx, AUTX_E_INVAL, "arrivals not in canonical order at index %u", i);
    } else if (prev && ctx->pend_set) {
      if (!std::lexicographical_compare(prev, prev + 4, key, key + 4))
        return fail(ctx, AUTX_E_INVAL, "arrivals not in canonical order across calls");
    }
    if (ctx->call_slot.count(d.call_id)) return fail(ctx, AUTX_E_EXIST, "duplicate call %llu", (unsigned long long)d.call_id);
    if (i > 0 && calls[i - 1].call_id == d.call_id) return fail(ctx, AUTX_E_EXIST, "duplicate call");
    uint64_t kvb0 = ((uint64_t)d.input_tokens + 1 + ctx->cfg.block_tokens - 1) / ctx->cfg.block_tokens;
    if (ctx->cfg.kv_budget_blocks != AUTX_INF && kvb0 > ctx->cfg.kv_budget_blocks)
      return fail(ctx, AUTX_E_INVAL, "call %llu needs %llu KV blocks > budget %u", (unsigned long long)d.call_id,
                  (unsigned long long)kvb0, ctx->cfg.kv_budget_blocks);
    if (!ctx->prog_row.count(d.program_id) && !new_prog_seen.count(d.program_id)) {
      new_prog_seen[d.program_id] = 1;
      ++new_progs;
    }
  }
  if (ctx->prog_free.size() + (ctx->cfg.max_programs - ctx->prog_next) < new_progs)
    return fail(ctx, AUTX_E_NOMEM, "process table full");
  // Eq. 2 parents: completed calls of the same, live program (validated before any mutation)
  uint32_t n_par = 0;
  if (poff) {
    if (poff[n] < poff[0]) return fail(ctx, AUTX_E_INVAL, "parent offsets not ascending");
    n_par = poff[n] - poff[0];
    if (n_par && !pids) return AUTX_E_INVAL;
    for (uint32_t i = 0; i < n; ++i) {
      if (poff[i + 1] < poff[i]) return fail(ctx, AUTX_E_INVAL, "parent offsets not ascending");
      if (poff[i + 1] - poff[i] >= (1u << 24)) return fail(ctx, AUTX_E_INVAL, "too many parents");
      const uint32_t* pr = ctx->prog_row.find(calls[i].program_id);
      for (uint32_t k = poff[i]; k < poff[i + 1]; ++k) {
        auto l = ctx->lin_of.find(pids[k]);
        if (l == ctx->lin_of.end())
          return fail(ctx, AUTX_E_NOENT, "parent %llu of call %llu is unknown", (unsigned long long)pids[k],
                      (unsigned long long)calls[i].call_id);
        if (ctx->call_slot.count(pids[k]))
          return fail(ctx, AUTX_E_STATE, "parent %llu of call %llu has not completed", (unsigned long long)pids[k],
                      (unsigned long long)calls[i].call_id);
        if (!pr || ctx->lin_prog[l->second] != *pr)
          return fail(ctx, AUTX_E_INVAL, "parent %llu of call %llu is in another program",
                      (unsigned long long)pids[k], (unsigned long long)calls[i].call_id);
      }
    }
  }
  if (ctx->eq2 && ctx->lin_free.size() + (ctx->lin_cap - ctx->lin_next) < n)
    return fail(ctx, AUTX_E_NOMEM, "Eq. 2 lineage capacity (%u) exhausted", ctx->lin_cap);
  if (ctx->n_par_staged + n_par > ctx->par_cap) {
    CK(cudaStreamSynchronize(ctx->stream));
    const uint32_t cap = std::max(ctx->n_par_staged + n_par, 2 * ctx->par_cap);
    uint32_t* nh = nullptr;
    CK(cudaHostAlloc((void**)&nh, (size_t)cap * 4, cudaHostAllocMapped));
    if (ctx->n_par_staged) memcpy(nh, ctx->h_par, (size_t)ctx->n_par_staged * 4);
    cudaFreeHost(ctx->h_par);
    ctx->h_par = nh;
    ctx->par_cap = cap;
  }
  if ((uint64_t)ctx->call_slot.size() + n > ctx->cfg.max_calls)
    return fail(ctx, AUTX_E_NOMEM, "call table full (%u active)", (unsigned)ctx->call_slot.size());
  if ((uint64_t)ctx->tail + n > ctx->cfg.max_calls) {
    s = flush_staged(ctx, t);  // staged rows must exist on the device before they move
    if (s) return s;
    s = compact(ctx);
    if (s) return s;
    // the flushed prologue (or its DMA) may still read the pinned staging this call refills
    CK(cudaStreamSynchronize(ctx->stream));
  }
  // staging buffer growth, keeping records already staged for this step
  const uint32_t need = ctx->n_arr_staged + n;
  if (need > ctx->arr_cap) {
    CK(cudaStreamSynchronize(ctx->stream));
    ArrivalRec* nh = nullptr;
    CK(cudaHostAlloc((void**)&nh, (size_t)need * sizeof(ArrivalRec), cudaHostAllocMapped));
    if (ctx->n_arr_staged) memcpy(nh, ctx->h_arr, (size_t)ctx->n_arr_staged * sizeof(ArrivalRec));
    cudaFreeHost(ctx->h_arr);
    cudaFree(ctx->d_arr);
    ctx->h_arr = nh;
    ctx->arr_cap = need;
    CK(dalloc(&ctx->d_arr, need));
  }
  if (ctx->n_arr_staged == 0) ctx->arr_first_slot = ctx->tail;
  ArrivalRec* stage = ctx->h_arr + ctx->n_arr_staged;
  // map program ids, build records
  for (uint32_t i = 0; i < n; ++i) {
    const autx_call_desc& d = calls[i];
    uint32_t flags = 0;
    const uint32_t* it = ctx->prog_row.find(d.program_id);
    uint32_t row;
    if (!it) {
      if (!ctx->prog_free.empty()) { row = ctx->prog_free.back(); ctx->prog_free.pop_back(); }
      else row = ctx->prog_next++;
      ctx->prog_row[d.program_id] = row;
      ctx->prog_active[row] = 0;
      CK(cudaMemsetAsync(ctx->d_pin + row, 0xff, 1, ctx->stream));
      flags = 3;  // new program, first record: the prologue zeroes its entry
      ctx->staged_new_progs.insert(d.program_id);
    } else {
      row = *it;
      // created earlier in this (not yet launched) step: inherit 0 without reading the entry
      if (ctx->staged_new_progs.count(d.program_id)) flags = 1;
    }
    ArrivalRec r{};
    r.cid = d.call_id;
    r.prog = row;
    r.tok = d.input_tokens;
    if (ctx->eq2) {
      uint32_t np = 0;
      if (poff) {
        np = poff[i + 1] - poff[i];
        r.par = ctx->n_par_staged;
        for (uint32_t k = poff[i]; k < poff[i + 1]; ++k) ctx->h_par[ctx->n_par_staged++] = ctx->lin_of[pids[k]];
      }
      flags |= np << 8;
      uint32_t L;
      if (!ctx->lin_free.empty()) { L = ctx->lin_free.back(); ctx->lin_free.pop_back(); }
      else L = ctx->lin_next++;
      ctx->lin_of[d.call_id] = L;
      ctx->lin_prog[L] = row;
      ctx->prog_calls[row].push_back(d.call_id);
    }
    r.flags = flags;
    stage[i] = r;
    uint32_t slot = ctx->tail + i;
    ctx->call_slot[d.call_id] = slot;
    ctx->slot_prog[slot] = row;
    ctx->slot_arr[slot] = t;
    ctx->slot_live[slot] = 1;
    ctx->prog_active[row] += 1;
  }
  const autx_call_desc& l = calls[n - 1];
  ctx->last_key[0] = l.arrival_step; ctx->last_key[1] = l.program_arrival_step;
  ctx->last_key[2] = l.program_id; ctx->last_key[3] = l.call_id;
  ctx->have_last_key = true;
  ctx->n_arr_staged += n;  // registered on the device by the next sched_step's prologue
  ctx->tail += n;
  ctx->n_reg_this += n;
  ctx->registered_this = true;
  ctx->pend_set = true;
  ctx->pend_t = t;
  return AUTX_OK;
}

// Replays the recorded launches of one step as a CUDA graph: the step is a launch-bound chain of
// a few small kernels, and one graph launch plus per-node parameter updates costs the host a
// fraction of the separate launches.  The graph of a new launch signature is captured once (with
// the PDL attribute, so consecutive kernel nodes keep their programmatic edges).
static autx_status step_graph_run(autx_ctx* ctx, std::vector<LaunchRec>& recs, size_t n_recs) {
  autx_ctx::StepGraph* sg = nullptr;
  for (auto& g : ctx->graphs) {
    bool same = g.funcs.size() == n_recs;
    for (size_t i = 0; same && i < n_recs; ++i)
      same = g.funcs[i] == recs[i].func && g.blocks[i].x == recs[i].block.x && g.smem[i] == recs[i].smem;
    if (same) { sg = &g; break; }
  }
  if (sg) {
    for (size_t i = 0; i < n_recs; ++i) {
      // only nodes whose parameters or grid changed: the chain reads the step's scalars from
      // the control block, so a typical step re-parameterises the prologue alone
      const dim3& g = recs[i].grid;
      if (sg->blobs[i] == recs[i].blob && sg->grids[i].x == g.x && sg->grids[i].y == g.y && sg->grids[i].z == g.z)
        continue;
      std::vector<void*> ptrs = recs[i].ptrs();
      cudaKernelNodeParams kp = {};
      kp.func = const_cast<void*>(recs[i].func);
      kp.gridDim = recs[i].grid;
      kp.blockDim = recs[i].block;
      kp.sharedMemBytes = (unsigned)recs[i].smem;
      kp.kernelParams = ptrs.data();
      CK(cudaGraphExecKernelNodeSetParams(sg->x, sg->nodes[i], &kp));
      sg->blobs[i] = recs[i].blob;
      sg->grids[i] = g;
    }
  } else {
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    if (ctx->graphs.size() >= 8) {  // bounded cache
      for (auto& g : ctx->graphs) { cudaGraphExecDestroy(g.x); cudaGraphDestroy(g.g); }
      ctx->graphs.clear();
    }
    autx_ctx::StepGraph g;
    CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t err = cudaSuccess;
    for (size_t ri = 0; ri < n_recs; ++ri) {
      LaunchRec& r = recs[ri];
      std::vector<void*> ptrs = r.ptrs();
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = r.grid;
      cfg.blockDim = r.block;
      cfg.dynamicSmemBytes = r.smem;
      cfg.stream = ctx->cap_stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      err = cudaLaunchKernelExC(&cfg, r.func, ptrs.data());
      if (err != cudaSuccess) break;
      cudaStreamCaptureStatus st;
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      err = cudaStreamGetCaptureInfo(ctx->cap_stream, &st, nullptr, nullptr, &deps, &nd);
      if (err != cudaSuccess || nd != 1) { if (err == cudaSuccess) err = cudaErrorUnknown; break; }
      g.nodes.push_back(deps[0]);
      g.funcs.push_back(r.func);
      g.blocks.push_back(r.block);
      g.smem.push_back(r.smem);
      g.blobs.push_back(r.blob);
      g.grids.push_back(r.grid);
    }
    cudaGraph_t graph = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(ctx->cap_stream, &graph);
    if (err != cudaSuccess || e2 != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      return fail(ctx, AUTX_E_CUDA, "step graph capture: %s", cudaGetErrorString(err != cudaSuccess ? err : e2));
    }
    g.g = graph;
    CK(cudaGraphInstantiate(&g.x, graph, 0));
    ctx->graphs.push_back(std::move(g));
    sg = &ctx->graphs.back();
  }
  CK(cudaGraphLaunch(sg->x, ctx->stream));
  return AUTX_OK;
}

extern "C" autx_status autx_sched_step(autx_ctx* ctx, uint32_t t, autx_step_out* out) {
  if (!ctx || !out) return AUTX_E_INVAL;
  g_hp.start();
  autx_status s = sync_last(ctx);
  if (s) return s;
  if (ctx->stepped && t <= ctx->t_last) return fail(ctx, AUTX_E_STATE, "step %u <= last step %u", t, ctx->t_last);
  if (ctx->pend_set && ctx->pend_t != t)
    return fail(ctx, AUTX_E_STATE, "registered arrivals are for step %u, not %u", ctx->pend_t, t);
  if (ctx->completed_this && t != next_step(ctx))
    return fail(ctx, AUTX_E_STATE, "completions are processed at step %u, not %u", next_step(ctx), t);
  if (ctx->stepped && t != ctx->t_last + 1 && ctx->call_slot.size() > ctx->n_reg_this)
    return fail(ctx, AUTX_E_STATE, "cannot skip steps while calls are active");
  if (ctx->cfg.nranks > 1 && !ctx->routed_this)
    return fail(ctx, AUTX_E_STATE, "multi-engine: autx_route_apply must run every step");
  // both orderings pack t - arrival (select: k_gather_ss / k_rank keys) or arrival - base (radix)
  // into a 27-bit key field
  while (ctx->low < ctx->tail && !ctx->slot_live[ctx->low]) ++ctx->low;
  const uint32_t arr_base = ctx->low < ctx->tail ? ctx->slot_arr[ctx->low] : t;
  if (t - arr_base >= (1u << 27)) return fail(ctx, AUTX_E_NOMEM, "arrival span exceeds the 27-bit key field");
  // the step's kernels as one graph replay (AUTX_NO_GRAPH: separate launches); not with the
  // per-kernel timing events, the radix pipeline (host-synchronised passes) or a bulk burst (DMA)
  static const bool no_graph = getenv("AUTX_NO_GRAPH") != nullptr;
  std::vector<LaunchRec>& recs = ctx->rec_pool;  // reused: no allocation per recorded launch
  const bool graph = !no_graph && !ctx->timing && !ctx->radix && ctx->n_arr_staged <= 4096;
  // R32: a window step keeps the resident list; the ordering runs at the first step, every N-th
  // step after the last scheduling point, and whenever the carried list is empty (the previous
  // step's resident calls, which the host knows from its record, minus this step's completions)
  bool window = false;
  if (ctx->pol.multistep) {
    const HostOut& h = *ctx->out.hout;
    const uint32_t carried = ctx->stepped ? h.n_batch + h.n_standby - (ctx->completed_this ? ctx->n_completed_pending : 0)
                                          : 0u;
    window = ctx->since != 0 && ctx->since < ctx->cfg.sched_every && carried > 0;
    ctx->since = window ? ctx->since + 1 : 1;
  }
  if (graph) { g_launch_rec = &recs; g_launch_n = 0; }
  ++ctx->seqno;
  g_hp.lap(0);
  s = flush_staged(ctx, t, true);  // the prologue, always: it hands t, n_rows, seqno to the chain
  if (s) { g_launch_rec = nullptr; return s; }
  g_hp.lap(1);
  const cudaError_t le = launch_step(ctx->stream, ctx->pol, ctx->ct, ctx->pt, ctx->ctl, ctx->out, ctx->kv,
                                     ctx->kv_on, t, ctx->tail, ctx->seqno, ctx->timing ? ctx->ev : nullptr,
                                     ctx->radix ? &ctx->rx : nullptr, arr_base, &ctx->radix_passes, window);
  g_launch_rec = nullptr;
  CK(le);
  g_hp.lap(2);
  if (graph) {
    s = step_graph_run(ctx, recs, g_launch_n);
    if (s) return s;
  }
  g_hp.lap(3);
  if (!ctx->out.zero_copy)
    CK(cudaMemcpyAsync(ctx->h_outblk, ctx->d_outblk, ctx->outblk_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaEventRecord(ctx->done, ctx->stream));
  ctx->pending_done = true;
  ctx->last_batch_valid = false;
  ctx->stepped = true;
  ctx->t_last = t;
  ctx->pend_set = false;
  ctx->completed_this = ctx->registered_this = false;
  ctx->routed_this = false;
  ctx->n_reg_this = 0;
  ctx->tc_step = ctx->timed_complete;
  ctx->tr_step = ctx->timed_register;
  ctx->timed_complete = ctx->timed_register = false;
  ctx->n_completed_pending = 0;
  ctx->have_last_key = false;
  memset(out, 0, sizeof *out);
  out->batch = ctx->out.batch_ids;
  out->admit = ctx->out.admit_ids;
  out->preempt = ctx->out.preempt_ids;
  out->h_batch = ctx->out.h_batch;
  out->h_admit = ctx->out.h_admit;
  out->h_preempt = ctx->out.h_preempt;
  out->done = (void*)ctx->done;
  g_hp.lap(4);
  ++g_hp.n;
  return AUTX_OK;
}

extern "C" autx_status autx_step_wait(autx_ctx* ctx, autx_step_out* out) {
  if (!ctx || !out) return AUTX_E_INVAL;
  autx_status s = sync_last(ctx);
  if (s) return s;
  const HostOut& h = *ctx->out.hout;
  if (h.seqno != ctx->seqno) return fail(ctx, AUTX_E_CUDA, "step output sequence mismatch");
  out->n_batch = h.n_batch;
  out->n_admit = h.n_admit;
  out->n_preempt = h.n_preempt;
  out->n_active = h.n_active;
  out->swap_out_blocks = h.swap_out_blocks;
  out->swap_in_blocks = h.swap_in_blocks;
  out->kv_blocks = h.kv_blocks;
  out->n_promoted = h.n_promoted;
  out->n_standby = h.n_standby;
  if (ctx->timing) {
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
    cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]);
    cudaEventElapsedTime(&c, ctx->ev[2], ctx->ev[3]);
    float d = 0, e = 0;
    if (ctx->tc_step) cudaEventElapsedTime(&d, ctx->ev[4], ctx->ev[5]);
    if (ctx->tr_step) cudaEventElapsedTime(&e, ctx->ev[6], ctx->ev[7]);
    ctx->last_timing.scan_ms = a;
    ctx->last_timing.select_ms = b;
    ctx->last_timing.finalize_ms = c;
    ctx->last_timing.complete_ms = d;
    ctx->last_timing.register_ms = e;
    ctx->last_timing.total_ms = a + b + c + d + e;
  }
  return AUTX_OK;
}

extern "C" autx_status autx_step(autx_ctx* ctx, uint32_t t, const uint64_t* completed, uint32_t n_completed,
                                 const uint64_t* ended_programs, uint32_t n_ended, const autx_call_desc* arrivals,
                                 uint32_t n_arrivals, autx_step_out* out) {
  if (!ctx || !out) return AUTX_E_INVAL;
  autx_status s = AUTX_OK;
  if (n_completed) s = autx_complete(ctx, completed, n_completed);
  for (uint32_t i = 0; s == AUTX_OK && i < n_ended; ++i) s = autx_end_program(ctx, ended_programs[i]);
  if (s == AUTX_OK && n_arrivals) s = autx_register_call(ctx, arrivals, n_arrivals);
  if (s == AUTX_OK) s = autx_sched_step(ctx, t, out);
  if (s == AUTX_OK) s = autx_step_wait(ctx, out);
  return s;
}

// G8: stable compaction on the device into the other half of the double-buffered call table
// (k_live_count, k_compact, k_remap_prev: no host sort, no allocation, no synchronisation).  The
// host remaps its own id maps in parallel: a live row's new index is its rank among the live rows,
// a prefix count over slot_live.
static autx_status compact(autx_ctx* ctx) {
  const uint32_t n = (uint32_t)ctx->call_slot.size();
  const auto t0 = std::chrono::steady_clock::now();
  CK(cudaMemsetAsync(ctx->ct2.qf, QF_DEAD, ctx->rows, ctx->stream));
  CK(launch_compact(ctx->stream, ctx->ct, ctx->ct2, ctx->tail, n, ctx->d_tile_live, ctx->d_old2new, ctx->ctl,
                    ctx->out.prev_slots));
  std::swap(ctx->ct, ctx->ct2);
  std::vector<uint32_t>& o2n = ctx->h_old2new;
  o2n.resize(std::max<uint32_t>(ctx->tail, 1));
  uint32_t k = 0;
  for (uint32_t r = 0; r < ctx->tail; ++r) {
    const bool live = ctx->slot_live[r];
    o2n[r] = live ? k : NONE;
    if (live) {
      ctx->slot_prog[k] = ctx->slot_prog[r];
      ctx->slot_arr[k] = ctx->slot_arr[r];
      ctx->slot_live[k] = 1;
      ++k;
    }
  }
  if (k != n) return fail(ctx, AUTX_E_STATE, "compaction: %u live rows on the host, %u active calls", k, n);
  std::fill(ctx->slot_live.begin() + k, ctx->slot_live.begin() + ctx->tail, 0);
  ctx->call_slot.for_each([&](uint64_t, uint32_t& v) { v = o2n[v]; });
  ctx->low = 0;
  ctx->tail = n;
  ++ctx->n_compactions;
  ctx->compact_host_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  return AUTX_OK;
}

// ---- KV swap ------------------------------------------------------------------------------
extern "C" autx_status autx_kv_swap(autx_ctx* ctx, const autx_kv_layout* L, int32_t mode,
                                    autx_swap_stats* stats) {
  if (!ctx || !L || !stats) return AUTX_E_INVAL;
  if (!ctx->kv_on) return fail(ctx, AUTX_E_INVAL, "KV allocator disabled (n_gpu_blocks == 0)");
  if (L->chunk_bytes % 16 || L->n_layers == 0 || !L->host_arena)
    return fail(ctx, AUTX_E_INVAL, "bad kv layout");
  uint64_t page = (uint64_t)L->n_layers * 2 * L->chunk_bytes;
  if (L->host_arena_bytes < ctx->cfg.host_pages * page)
    return fail(ctx, AUTX_E_INVAL, "host arena smaller than host_pages * page bytes");
  autx_status s = sync_last(ctx);
  if (s) return s;
  if (2 * L->n_layers > ctx->pools_cap) {
    if (ctx->d_pools) cudaFree(ctx->d_pools);
    if (ctx->h_pools) cudaFreeHost(ctx->h_pools);
    ctx->pools_cap = 2 * L->n_layers;
    CK(dalloc(&ctx->d_pools, ctx->pools_cap));
    CK(cudaHostAlloc((void**)&ctx->h_pools, ctx->pools_cap * sizeof(void*), 0));
  }
  CK(cudaStreamSynchronize(ctx->stream));  // h_pools reuse
  for (uint32_t l = 0; l < L->n_layers; ++l) {
    ctx->h_pools[l] = L->k_pool[l];
    ctx->h_pools[L->n_layers + l] = L->v_pool[l];
  }
  CK(cudaMemcpyAsync(ctx->d_pools, ctx->h_pools, 2 * L->n_layers * sizeof(void*), cudaMemcpyHostToDevice,
                     ctx->stream));
  Ctl c;
  CK(cudaMemcpyAsync(&c, ctx->ctl, sizeof c, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  memset(stats, 0, sizeof *stats);
  stats->bytes_d2h = (uint64_t)c.plan_out_chunks * page;
  stats->bytes_h2d = (uint64_t)c.plan_in_chunks * page;
  stats->chunks_d2h = c.plan_out_chunks * L->n_layers * 2;
  stats->chunks_h2d = c.plan_in_chunks * L->n_layers * 2;
  void** kp = ctx->d_pools;
  void** vp = ctx->d_pools + L->n_layers;
  char* arena = (char*)L->host_arena;
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, ctx->device);
  CK(cudaEventRecord(ctx->sev[0], ctx->stream));
  // full duplex: both directions at once unless a swap-in target block was freed by this step's
  // swap-out (the allocator avoids that while older free blocks last; ctl->swap_serial)
  // (the per-chunk comparator stays vLLM's: one stream, one copy at a time)
  const bool duplex = c.plan_out_chunks && c.plan_in_chunks && !c.swap_serial && mode != AUTX_SWAP_PER_CHUNK_MEMCPY &&
                      !getenv("AUTX_SWAP_HALF_DUPLEX");
  ctx->last_swap_duplex = duplex;
  if (mode == AUTX_SWAP_SM) {
    if (duplex) {
      CK(launch_swap(ctx->stream, ctx->ctl, ctx->kv, kp, vp, L->n_layers, L->chunk_bytes, arena, 2, dev_sms * 8));
    } else {
      if (c.plan_out_chunks) CK(launch_swap(ctx->stream, ctx->ctl, ctx->kv, kp, vp, L->n_layers, L->chunk_bytes, arena, 0, dev_sms * 4));
      if (c.plan_in_chunks) CK(launch_swap(ctx->stream, ctx->ctl, ctx->kv, kp, vp, L->n_layers, L->chunk_bytes, arena, 1, dev_sms * 4));
    }
  } else if (mode == AUTX_SWAP_PER_CHUNK_MEMCPY || mode == AUTX_SWAP_STAGED_DMA) {
    // both comparators need the plan on the host
    std::vector<PlanItem> po(c.n_plan_out), pi(c.n_plan_in);
    std::vector<uint32_t> bo(c.plan_out_chunks), bi(c.plan_in_chunks);
    if (c.n_plan_out) CK(cudaMemcpy(po.data(), ctx->kv.plan_out, po.size() * sizeof(PlanItem), cudaMemcpyDeviceToHost));
    if (c.n_plan_in) CK(cudaMemcpy(pi.data(), ctx->kv.plan_in, pi.size() * sizeof(PlanItem), cudaMemcpyDeviceToHost));
    if (c.plan_out_chunks) CK(cudaMemcpy(bo.data(), ctx->kv.plan_out_blocks, bo.size() * 4, cudaMemcpyDeviceToHost));
    if (c.plan_in_chunks) CK(cudaMemcpy(bi.data(), ctx->kv.plan_in_blocks, bi.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaEventRecord(ctx->sev[0], ctx->stream));
    if (mode == AUTX_SWAP_PER_CHUNK_MEMCPY) {
      // vLLM v0.6.1 behaviour: one cudaMemcpyAsync per (layer, K|V, block)
      for (int dir = 0; dir < 2; ++dir) {
        auto& items = dir == 0 ? po : pi;
        auto& blks = dir == 0 ? bo : bi;
        for (auto& it : items)
          for (uint32_t j = 0; j < it.nblk; ++j)
            for (uint32_t l = 0; l < L->n_layers; ++l)
              for (int kvs = 0; kvs < 2; ++kvs) {
                char* dev = (char*)(kvs ? L->v_pool[l] : L->k_pool[l]) + (uint64_t)blks[it.blk_off + j] * L->chunk_bytes;
                char* host = arena + it.host_page * page + ((uint64_t)j * L->n_layers + l) * 2 * L->chunk_bytes +
                             (uint64_t)kvs * L->chunk_bytes;
                if (dir == 0) CK(cudaMemcpyAsync(host, dev, L->chunk_bytes, cudaMemcpyDeviceToHost, ctx->stream));
                else CK(cudaMemcpyAsync(dev, host, L->chunk_bytes, cudaMemcpyHostToDevice, ctx->stream));
              }
      }
    } else {
      // the paper's scheme: gather into a contiguous buffer, one bulk transfer
      // per call
      auto grow = [&](char** buf, size_t* have, size_t need) -> cudaError_t {
        if (need <= *have) return cudaSuccess;
        if (*buf) cudaFree(*buf);
        *buf = nullptr;
        *have = 0;
        cudaError_t e = cudaMalloc((void**)buf, need);
        if (e == cudaSuccess) *have = need;
        return e;
      };
      const size_t need_out = (size_t)c.plan_out_chunks * page, need_in = (size_t)c.plan_in_chunks * page;
      if (need_out > ctx->staging_bytes || need_in > (duplex ? ctx->staging_in_bytes : ctx->staging_bytes)) {
        CK(grow(&ctx->staging, &ctx->staging_bytes, duplex ? need_out : std::max(need_out, need_in)));
        if (duplex) CK(grow(&ctx->staging_in, &ctx->staging_in_bytes, need_in));
        CK(cudaEventRecord(ctx->sev[0], ctx->stream));  // (allocations synchronise: time from here)
      }
      // swap-in leg: on its own stream when the directions may overlap (both copy engines and
      // both link directions busy at once), after everything before this call on ctx->stream
      cudaStream_t sin = ctx->stream;
      char* st_in = ctx->staging;
      if (duplex) {
        if (!ctx->stream_in) {
          CK(cudaStreamCreateWithFlags(&ctx->stream_in, cudaStreamNonBlocking));
          CK(cudaEventCreateWithFlags(&ctx->sev_in[0], cudaEventDisableTiming));
          CK(cudaEventCreateWithFlags(&ctx->sev_in[1], cudaEventDisableTiming));
        }
        CK(cudaEventRecord(ctx->sev_in[0], ctx->stream));
        CK(cudaStreamWaitEvent(ctx->stream_in, ctx->sev_in[0], 0));
        sin = ctx->stream_in;
        st_in = ctx->staging_in;
      }
      if (c.plan_out_chunks) {
        CK(launch_stage(ctx->stream, ctx->ctl, ctx->kv, kp, vp, L->n_layers, L->chunk_bytes, ctx->staging, 0, dev_sms * 4));
        for (auto& it : po)
          CK(cudaMemcpyAsync(arena + it.host_page * page, ctx->staging + (uint64_t)it.blk_off * page,
                             (uint64_t)it.nblk * page, cudaMemcpyDeviceToHost, ctx->stream));
      }
      if (c.plan_in_chunks) {
        for (auto& it : pi)
          CK(cudaMemcpyAsync(st_in + (uint64_t)it.blk_off * page, arena + it.host_page * page,
                             (uint64_t)it.nblk * page, cudaMemcpyHostToDevice, sin));
        CK(launch_stage(sin, ctx->ctl, ctx->kv, kp, vp, L->n_layers, L->chunk_bytes, st_in, 1, dev_sms * 4));
      }
      if (duplex) {
        CK(cudaEventRecord(ctx->sev_in[1], sin));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->sev_in[1], 0));
      }
    }
  } else {
    return fail(ctx, AUTX_E_INVAL, "unknown swap mode %d", mode);
  }
  CK(cudaEventRecord(ctx->sev[1], ctx->stream));
  CK(cudaEventSynchronize(ctx->sev[1]));
  CK(cudaEventElapsedTime(&stats->ms, ctx->sev[0], ctx->sev[1]));
  stats->duplex = ctx->last_swap_duplex ? 1u : 0u;
  return AUTX_OK;
}

extern "C" autx_status autx_block_table(autx_ctx* ctx, const uint32_t** off, const uint32_t** blk) {
  if (!ctx || !off || !blk) return AUTX_E_INVAL;
  if (!ctx->kv_on) return fail(ctx, AUTX_E_INVAL, "KV allocator disabled");
  *off = ctx->kv.bt_offsets;
  *blk = ctx->kv.bt_blocks;
  return AUTX_OK;
}

extern "C" autx_status autx_block_table_host(autx_ctx* ctx, uint32_t* h_off, uint32_t* h_blk, uint32_t cap,
                                             uint32_t* n_batch) {
  if (!ctx || !h_off || !n_batch) return AUTX_E_INVAL;
  if (!ctx->kv_on) return fail(ctx, AUTX_E_INVAL, "KV allocator disabled");
  autx_status s = sync_last(ctx);
  if (s) return s;
  CK(cudaStreamSynchronize(ctx->stream));
  uint32_t n = ctx->out.hout->n_batch;
  CK(cudaMemcpy(h_off, ctx->kv.bt_offsets, (size_t)(n + 1) * 4, cudaMemcpyDeviceToHost));
  uint32_t nb = h_off[n];
  if (nb > cap) return fail(ctx, AUTX_E_INVAL, "block table needs %u entries", nb);
  if (nb) CK(cudaMemcpy(h_blk, ctx->kv.bt_blocks, (size_t)nb * 4, cudaMemcpyDeviceToHost));
  *n_batch = n;
  return AUTX_OK;
}

// ---- introspection ---------------------------------------------------------------------------
extern "C" autx_status autx_dump_calls(autx_ctx* ctx, autx_call_state* outp, uint32_t cap, uint32_t* n) {
  if (!ctx || !n) return AUTX_E_INVAL;
  autx_status s = sync_last(ctx);
  if (s) return s;
  CK(cudaStreamSynchronize(ctx->stream));
  uint32_t T = ctx->tail;
  std::vector<uint64_t> cid(T);
  std::vector<uint32_t> arr(T), base(T), mt(T), ex(T), qt(T), inh(T), tok(T);
  std::vector<uint8_t> qf(T);
  const CallTable& t = ctx->ct;
  if (T) {
    CK(cudaMemcpy(cid.data(), t.cid, (size_t)T * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(arr.data(), t.arr, (size_t)T * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(base.data(), t.base, (size_t)T * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(mt.data(), t.mtime, (size_t)T * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ex.data(), t.exec, (size_t)T * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(qt.data(), t.quanta, (size_t)T * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(inh.data(), t.inh, (size_t)T * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tok.data(), t.tok, (size_t)T * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(qf.data(), t.qf, T, cudaMemcpyDeviceToHost));
  }
  const uint32_t now = ctx->stepped ? ctx->t_last + 1 : 0;  // counters include step t_last
  uint32_t k = 0;
  for (uint32_t r = 0; r < T; ++r) {
    if (qf[r] & QF_DEAD) continue;
    if (outp && k < cap) {
      autx_call_state& o = outp[k];
      o.call_id = cid[r];
      o.q = qf[r] & QF_QMASK;
      o.quanta = qt[r];
      o.mtime = mt[r];
      o.wait = (now - base[r]) - mt[r];
      o.exec = ex[r];
      o.totwait = (now - arr[r]) - ex[r];
      o.inh = inh[r];
      o.input_tokens = tok[r];
      o.arrival_step = arr[r];
      o.flags = ((qf[r] & QF_RUN) ? 1u : 0u) | ((qf[r] & QF_RES) ? 2u : 0u) |
                ((!(qf[r] & QF_RES) && ex[r] > 0) ? 4u : 0u);
    }
    ++k;
  }
  *n = k;
  return AUTX_OK;
}

extern "C" autx_status autx_program_state(autx_ctx* ctx, uint64_t pid, uint32_t* svc, uint64_t* pwait) {
  if (!ctx) return AUTX_E_INVAL;
  const uint32_t* it = ctx->prog_row.find(pid);
  if (!it) return fail(ctx, AUTX_E_NOENT, "unknown program");
  CK(cudaStreamSynchronize(ctx->stream));
  PInfo pi;
  CK(cudaMemcpy(&pi, ctx->pt.info + *it, sizeof pi, cudaMemcpyDeviceToHost));
  if (svc) *svc = pi.svc;
  if (pwait) *pwait = pi.pwait;
  return AUTX_OK;
}

extern "C" autx_status autx_step_stats(autx_ctx* ctx, autx_selection_stats* o) {
  if (!ctx || !o) return AUTX_E_INVAL;
  autx_status s = sync_last(ctx);
  if (s) return s;
  CK(cudaStreamSynchronize(ctx->stream));
  Ctl c;
  CK(cudaMemcpy(&c, ctx->ctl, sizeof c, cudaMemcpyDeviceToHost));
  memset(o, 0, sizeof *o);
  o->qstar = c.qstar;
  o->mprime = c.mprime;
  o->n_x = c.n_cand_a;
  o->n_b = c.last_n_b;
  o->n_rows = ctx->tail;
  o->n_programs = (uint32_t)ctx->prog_row.size();
  if (!ctx->radix && ctx->stepped) {
    const uint32_t ntiles = std::max<uint32_t>(1, (ctx->tail + TILE - 1) / TILE);
    std::vector<uint32_t> cnt((size_t)ntiles * MAX_K);
    CK(cudaMemcpy(cnt.data(), ctx->out.tile_cnt, cnt.size() * 4, cudaMemcpyDeviceToHost));
    for (uint32_t t = 0; t < ntiles; ++t)
      for (int k = 0; k < MAX_K; ++k) o->queue_counts[k] += cnt[(size_t)t * MAX_K + k];
  }
  return AUTX_OK;
}

extern "C" autx_status autx_last_step_timing(autx_ctx* ctx, autx_step_timing* t) {
  if (!ctx || !t) return AUTX_E_INVAL;
  *t = ctx->last_timing;
  return AUTX_OK;
}

extern "C" autx_status autx_set_timing(autx_ctx* ctx, int32_t on) {
  if (!ctx) return AUTX_E_INVAL;
  ctx->timing = (on & 1) != 0;       // 1: CUDA events around the step's kernels
  ctx->pol.stamps = (on & 2) ? 1 : 0;  // 2: %globaltimer chain stamps (no events: PDL undisturbed)
  return AUTX_OK;
}

extern "C" autx_status autx_compaction_stats(const autx_ctx* ctx, uint64_t* n, double* host_us) {
  if (!ctx || !n || !host_us) return AUTX_E_INVAL;
  *n = ctx->n_compactions;
  *host_us = ctx->compact_host_us;
  return AUTX_OK;
}

extern "C" uint32_t autx_num_active(const autx_ctx* ctx) { return ctx ? (uint32_t)ctx->call_slot.size() : 0; }

// ---- routing (a8) ----------------------------------------------------------------------------
extern "C" uint64_t autx_route_record_bytes(const autx_ctx* ctx) {
  return ctx ? sizeof(RouteHdr) + (uint64_t)ctx->cfg.max_batch * sizeof(CompRec) : 0;
}

extern "C" autx_status autx_route_pack(autx_ctx* ctx, void* d_record) {
  if (!ctx || !d_record) return AUTX_E_INVAL;
  autx_status s = sync_last(ctx);
  if (s) return s;
  if (ctx->registered_this) return fail(ctx, AUTX_E_STATE, "autx_route_pack after autx_register_call");
  // header from the kernel parameters (queued + running after this step's completions, R21)
  const uint32_t n_comp = ctx->completed_this ? ctx->n_completed_pending : 0;
  CK(launch_route_hdr(ctx->stream, d_record, ctx->call_slot.size(), n_comp));
  if (n_comp)
    CK(cudaMemcpyAsync((char*)d_record + sizeof(RouteHdr), ctx->d_route_local + sizeof(RouteHdr),
                       (size_t)n_comp * sizeof(CompRec), cudaMemcpyDeviceToDevice, ctx->stream));
  return AUTX_OK;
}

// Steps 3-4 of a routing epoch over the gathered records (d_records: nranks records of
// autx_route_record_bytes() each): apply every engine's completion records, then Alg. 2.
static autx_status route_common(autx_ctx* ctx, const void* d_records, const autx_call_desc* calls, uint32_t n,
                                int32_t* engine_out) {
  const uint32_t G = (uint32_t)std::max(ctx->cfg.nranks, 1);
  const uint32_t t = next_step(ctx);
  const uint64_t stride = autx_route_record_bytes(ctx);
  if (ctx->cfg.nranks > 1) CK(launch_apply(ctx->stream, ctx->pol, ctx->pt, d_records, stride, G, t));
  if (n > ctx->rarr_cap) {
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->h_rarr) cudaFreeHost(ctx->h_rarr);
    if (ctx->d_rarr) cudaFree(ctx->d_rarr);
    if (ctx->d_rout) cudaFree(ctx->d_rout);
    ctx->rarr_cap = n;
    CK(cudaHostAlloc((void**)&ctx->h_rarr, (size_t)n * sizeof(RouteArr), 0));
    CK(dalloc(&ctx->d_rarr, n));
    CK(dalloc(&ctx->d_rout, n));
  }
  // (h_rarr is free to refill: the last epoch that used it synchronised on its engine_out copy)
  // replicated process-table rows: created in canonical arrival order on every rank
  for (uint32_t i = 0; i < n; ++i) {
    const autx_call_desc& d = calls[i];
    if (i > 0) {
      const autx_call_desc& q = calls[i - 1];
      uint64_t a[4] = {q.arrival_step, q.program_arrival_step, q.program_id, q.call_id};
      uint64_t b[4] = {d.arrival_step, d.program_arrival_step, d.program_id, d.call_id};
      if (!std::lexicographical_compare(a, a + 4, b, b + 4))
        return fail(ctx, AUTX_E_INVAL, "routing batch not in canonical order");
    }
    const uint32_t* it = ctx->prog_row.find(d.program_id);
    uint32_t row;
    if (!it) {
      autx_status s2 = new_program(ctx, d.program_id, &row);
      if (s2) return s2;
    } else {
      row = *it;
    }
    ctx->h_rarr[i] = RouteArr{row, d.input_tokens};
  }
  if (n) {
    CK(cudaMemcpyAsync(ctx->d_rarr, ctx->h_rarr, (size_t)n * sizeof(RouteArr), cudaMemcpyHostToDevice, ctx->stream));
    CK(launch_route(ctx->stream, d_records, stride, G, ctx->d_rarr, n, ctx->d_pin, ctx->cfg.token_threshold,
                    ctx->d_rout, ctx->cfg.route_policy, ctx->d_rr));
    CK(cudaMemcpyAsync(engine_out, ctx->d_rout, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  ctx->routed_this = true;
  return AUTX_OK;
}

static autx_status route_checks(autx_ctx* ctx, const autx_call_desc* calls, uint32_t n, int32_t* engine_out) {
  if (n && (!calls || !engine_out)) return fail(ctx, AUTX_E_INVAL, "calls / engine_out");
  if (ctx->registered_this) return fail(ctx, AUTX_E_STATE, "routing after autx_register_call");
  if (ctx->routed_this) return fail(ctx, AUTX_E_STATE, "routing twice in one step");
  return AUTX_OK;
}

extern "C" autx_status autx_route_apply(autx_ctx* ctx, const void* d_records, const autx_call_desc* calls,
                                        uint32_t n, int32_t* engine_out) {
  if (!ctx || !d_records) return AUTX_E_INVAL;
  if (autx_status s = route_checks(ctx, calls, n, engine_out)) return s;
  return route_common(ctx, d_records, calls, n, engine_out);
}

#define NCK(call)                                                                                  \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess) return fail(ctx, AUTX_E_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

extern "C" autx_status autx_route(autx_ctx* ctx, const autx_call_desc* calls, uint32_t n, int32_t* engine_out) {
  if (!ctx) return AUTX_E_INVAL;
  if (autx_status s = route_checks(ctx, calls, n, engine_out)) return s;
  const int G = std::max(ctx->cfg.nranks, 1);
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(ctx->cfg.nccl_comm);
  if (G > 1 && !comm) return fail(ctx, AUTX_E_INVAL, "autx_route with nranks > 1 needs autx_config.nccl_comm");
  autx_status s = sync_last(ctx);  // the previous step's host-visible state (no device wait otherwise)
  if (s) return s;
  // 1. this engine's epoch record: header from the host's counts, records already on the device
  //    (written by autx_complete's kernel)
  const uint32_t n_comp = ctx->completed_this ? ctx->n_completed_pending : 0;
  CK(launch_route_hdr(ctx->stream, ctx->d_route_local, ctx->call_slot.size(), n_comp));
  // 2. the all-gather of the fixed-size records, stream-ordered (NCCL over NVLink / NVSwitch)
  const size_t stride = autx_route_record_bytes(ctx);
  const void* recs = ctx->d_route_local;
  if (comm) {
    int cr = 0, cn = 0;
    NCK(ncclCommCount(comm, &cn));
    NCK(ncclCommUserRank(comm, &cr));
    if (cn != G || cr != ctx->cfg.rank)
      return fail(ctx, AUTX_E_INVAL, "nccl_comm is rank %d of %d, config says %d of %d", cr, cn, ctx->cfg.rank, G);
    NCK(ncclAllGather(ctx->d_route_local, ctx->d_route_all, stride, ncclUint8, comm, ctx->stream));
    recs = ctx->d_route_all;
  }
  // 3-4. apply every engine's records, route with Alg. 2
  return route_common(ctx, recs, calls, n, engine_out);
}

extern "C" autx_status autx_comm_unique_id(void* id_out) {
  if (!id_out) return AUTX_E_INVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return AUTX_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id_out, &id, sizeof id);
  return AUTX_OK;
}

extern "C" autx_status autx_comm_init(const void* id, int32_t rank, int32_t nranks, int32_t device, void** comm_out) {
  if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return AUTX_E_INVAL;
  *comm_out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return AUTX_E_CUDA;
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  ncclComm_t c = nullptr;
  if (ncclCommInitRank(&c, nranks, u, rank) != ncclSuccess) return AUTX_E_NCCL;
  *comm_out = c;
  return AUTX_OK;
}

extern "C" autx_status autx_comm_destroy(void* comm) {
  if (!comm) return AUTX_E_INVAL;
  return ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm)) == ncclSuccess ? AUTX_OK : AUTX_E_NCCL;
}

extern "C" autx_status autx_phase_times(autx_ctx* ctx, uint64_t* ns, uint32_t cap) {
  if (!ctx || !ns) return AUTX_E_INVAL;
  CK(cudaStreamSynchronize(ctx->stream));
  Ctl c;
  CK(cudaMemcpy(&c, ctx->ctl, sizeof c, cudaMemcpyDeviceToHost));
  memcpy(ns, c.dbg, std::min<uint32_t>(cap, 96) * 8);
  return AUTX_OK;
}
