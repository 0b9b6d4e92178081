#!/usr/bin/env python
"""Benchmark of the Autellix scheduler hot path on B200 (BASELINE.json metric:
"sched decisions/s at 1M active calls; KV swap GB/s; % roofline at 1/2/4/8 GPUs").

A step = one pass of SURVEY §8(a) rows a1-a6 (+ a8 when N > 1) through the C ABI over the
whole active set: completions of the previous step, arrivals, demotion, anti-starvation,
ordering, cutoff, admit/preempt lists and accounting.  In select mode the device work of a step
is ONE cooperative kernel (k_step).  Workload (BASELINE configs[3], the default): an offline
burst of 50/50 LATS-MCTS and map-reduce DAG programs with ~1M calls ready at step 0,
ATLAS, SPEC ladder (K=8), beta=2, BS=1024, KV budget 32768 blocks of 16 tokens, fast-forwarded
10,000 steps so that queues, waits and promotions are diverse; decisions/s = active calls ranked
per step / device step time.  Other workloads: --workload mixed4m (configs[4] on one engine: 4M
calls, beyond L2), chatbot / react (configs[1] / [2]), churn (about BS completions and BS
arrivals per step).  The KV swap (row a7) is timed in a second phase on the ReAct-shaped config
with 8B-geometry pools (32 layers x 32 KiB chunks) and reported under "swap".

Timing: W warm-up steps, then K steps; before each step L2 is flushed (a 512 MiB write) and a
spin kernel gates the stream while the host enqueues the step, so CUDA events around the step
measure device time only.  Multi-GPU: one rank per GPU (torchrun), each rank runs its own
shard; every step includes the routing epoch (completion records + load all-gathered over NCCL,
Alg. 2 over the replicated arrivals).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
# SURVEY §8(d) algorithmic bytes of one step: per active call 34 B read (prog, arr, seq, q,
# flags, quanta, wait, mtime, exec, kvb) + 18 B written (q, flags, quanta, wait, mtime, exec);
# per program 16 B (svc, pwait, parr, pin).  The roofline fraction uses these.
ALGO_BYTES_PER_CALL = 52
ALGO_BYTES_PER_PROGRAM = 16
# What this design actually has to stream per step: the dense pass reads qf 1 +
# prog 4 + base 4 + mtime 4 per row and the program rows it gathers (svc 4 + pwait 8).
DESIGN_BYTES_PER_ROW = 13
DESIGN_BYTES_PER_PROGRAM = 12


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="autx", choices=["autx", "reference"])
    ap.add_argument("--active", type=int, default=None, help="active calls of the burst (workload default)")
    ap.add_argument("--ff", type=int, default=10_000, help="fast-forward steps before warm-up")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-swap", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--swap-steps", type=int, default=60)
    ap.add_argument("--order", default="select", choices=["select", "radix"])
    ap.add_argument("--beta", default="2", choices=["2", "inf"], help="anti-starvation threshold")
    ap.add_argument("--policy", default=None, choices=["atlas", "atlas_eq2", "plas"],
                    help="override the workload's policy (atlas_eq2: exact Eq. 2, SURVEY 8(f) item 2)")
    ap.add_argument("--workload", default="mcts", choices=list(WORKLOADS),
                    help="mcts: BASELINE configs[3] (default, the headline); mixed4m: configs[4] on one "
                         "engine; chatbot/react: configs[1]/[2]; churn: ~BS completions + arrivals per step")
    ap.add_argument("--json-out", default=None, help="also write the JSON line to this file")
    return ap.parse_args()


WORKLOADS = {
    "mcts": dict(policy="atlas", max_batch=1024, kv_budget=32768, active=1_000_000,
                 desc="mcts_mapreduce_burst (BASELINE configs[3])"),
    "mixed4m": dict(policy="atlas", max_batch=1024, kv_budget=32768, active=4_000_000,
                    desc="mixed burst, equal draw chat / ReAct / MCTS+map-reduce (BASELINE configs[4] on one engine)"),
    "chatbot": dict(policy="plas", max_batch=256, kv_budget=6000, active=10_000,
                    desc="chatbot 10k ShareGPT-shaped programs (BASELINE configs[1])"),
    "react": dict(policy="plas", max_batch=256, kv_budget=8000, active=100_000,
                  desc="ReAct 100k BFCL-shaped programs (BASELINE configs[2])"),
    "churn": dict(policy="atlas", max_batch=1024, kv_budget=None, active=1_000_000,
                  desc="churn stress: 1M one-token chains, ~BS completions and BS arrivals per step"),
}


def make_trace(name, active, seed_off=0):
    from autx_workload import (burst_mcts_mapreduce, burst_mixed, chatbot, react, churn, BASE_SEED,
                               CONFIG_INDEX)
    if name == "mcts":
        return burst_mcts_mapreduce(active, seed=BASE_SEED + CONFIG_INDEX["mcts"] + seed_off)
    if name == "mixed4m":
        return burst_mixed(active, seed=BASE_SEED + CONFIG_INDEX["multi"] + seed_off)
    if name == "chatbot":
        return chatbot(active, seed=BASE_SEED + CONFIG_INDEX["chatbot"] + seed_off)
    if name == "react":
        return react(active, seed=BASE_SEED + CONFIG_INDEX["react"] + seed_off)
    return churn(active, seed=BASE_SEED + 100 + seed_off)


CHAIN = ["prologue", "scan", "select", "gather", "rank", "finalize"]


def chain_spans(phase):
    """Median (CTA 0 past griddepcontrol.wait, latest CTA end, latest CTA past the wait) in us of
    each kernel of the step chain, relative to the first kernel's CTA 0, from the library's
    %globaltimer chain stamps (autx_set_timing mode 2: autx_phase_times [64, 96))."""
    rows = []
    for p in phase:
        c = [int(x) for x in p[64:96]]
        starts = [c[3 * k] for k in range(6) if c[3 * k]]
        if not starts:
            continue
        t0 = min(starts)
        rows.append({n: (c[3 * k] - t0, c[3 * k + 1] - t0, c[3 * k + 2] - t0) for k, n in enumerate(CHAIN)
                     if c[3 * k]})
    out = {}
    for n in CHAIN:
        v = [r[n] for r in rows if n in r]
        if v:
            out[n] = [round(float(np.median([x[i] for x in v])) / 1e3, 2) for i in range(3)]
    return out or None


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of one step's kernels (summed over the chain)
    from the committed `ncu --set full` capture summary (profiles/step_traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "step_traffic.json")))
        return d["dram_bytes_per_launch"], d.get("source")
    except Exception:
        return None, None


def peaks():
    try:
        d = json.load(open(MEASURED_PEAKS))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def spec_ladder():
    """SPEC default ladder: K=8, hi_i = 2*4^(i-1), quanta = band widths."""
    hi = tuple(2 * 4 ** i for i in range(7))
    lo = (0,) + hi
    quanta = tuple(hi[i] - lo[i] for i in range(7)) + (None,)
    return dict(K=8, q_hi=hi, quanta=quanta)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, path):
        self.path = path
        self.p = None

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self, device=0):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or f[0] != str(device):
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_init(n):
    import torch
    import torch.distributed as dist
    if n <= 1 or "RANK" not in os.environ:
        return 0, 1, 0
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if os.environ.get("AUTX_DIST_BACKEND", "nccl") == "gloo":   # tests: several ranks on one GPU
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


# ------------------------------------------------------------------------------------------
# reference arm: the CPU oracle as it stands, on a bounded sample of the same workload
# ------------------------------------------------------------------------------------------
def oracle_decisions_per_s(active, steps, warmup, seed_off=0):
    from autx_workload import burst_mcts_mapreduce, BASE_SEED, CONFIG_INDEX
    from oracle.autellix import Engine, Workload, Config
    lad = spec_ladder()
    tr = burst_mcts_mapreduce(active, seed=BASE_SEED + CONFIG_INDEX["mcts"] + seed_off)
    cfg = Config(policy="atlas", beta=(2, 1), max_batch=1024, kv_budget=32768, **lad)
    eng = Engine(cfg, check_formulations=False)
    wl = Workload(tr)
    completed = []
    times, decisions = [], 0
    t0 = time.perf_counter()
    for t in range(1 + warmup + steps):
        cids = [int(tr.call_id[c]) for c in completed]
        ended = wl.release(t, completed)
        s = time.perf_counter()
        rec = eng.step(t, cids, wl.arrivals(t))
        dt = time.perf_counter() - s
        for pid in ended:
            eng.table.end_program(pid)
        completed = wl.ran(t, rec["batch"])
        if t > warmup:  # step 0 registers the whole burst: setup, not timed
            times.append(dt)
            decisions += rec["n_active"]
    return decisions / sum(times), sum(times) / len(times), time.perf_counter() - t0, tr.n_calls


def run_reference(args, rank, world):
    if rank != 0:
        return
    active = max(10_000, (args.active or 1_000_000) // 10)
    steps = max(1, min(args.steps, 10))
    v, per_step, wall, _ = oracle_decisions_per_s(active, steps, min(args.warmup, 3))
    line = {"metric": "sched decisions/s at 1M active calls", "value": v, "unit": "decisions/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": min(args.warmup, 3),
            "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "mcts_mapreduce_burst", "active_calls": active, "policy": "atlas",
                       "max_batch": 1024, "kv_budget_blocks": 32768, "sample": "1/10 of the 1M burst"},
            "cpu_baseline": {"value": v, "unit": "decisions/s", "cores": 1, "kind": "oracle",
                             "sample": f"{active}-call burst (1/10 of the 1M config), {steps} steps after setup"},
            "e2e": {"value": v, "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# KV swap phase (row a7)
# ------------------------------------------------------------------------------------------
def host_link_peak(torch, nbytes=1 << 30):
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    res = {}
    for name, (dst, src) in {"d2h": (host, dev), "h2d": (dev, host)}.items():
        best = 0.0
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dst.copy_(src, non_blocking=True)
            b.record()
            b.synchronize()
            best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
        res[name] = best
    # both directions at once, on two streams (two copy engines, both halves of the link)
    dev2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    host2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = 0.0
    for _ in range(5):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b1, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s1.wait_event(a)
        s2.wait_event(a)
        with torch.cuda.stream(s1):
            host.copy_(dev, non_blocking=True)
            b1.record(s1)
        with torch.cuda.stream(s2):
            dev2.copy_(host2, non_blocking=True)
            b2.record(s2)
        b1.synchronize()
        b2.synchronize()
        ms = max(a.elapsed_time(b1), a.elapsed_time(b2))
        best = max(best, 2 * nbytes / (ms * 1e-3) / 1e9)
    res["duplex"] = best
    del dev, host, dev2, host2
    return res


def bench_swap(torch, args, link):
    """Row a7 on the ReAct-shaped config with 8B-geometry pools, three modes.  Every run also
    checks the swapped bytes (SURVEY §8(d) "pattern round trip on every benchmark run"): the
    "engine" fills each newly allocated block of a call with a pattern of (call, block, layer,
    K|V) in every layer, and every block a call gets back after a swap-out / swap-in round trip
    (possibly another GPU block id) must hold its pattern, in all 32 layers x K|V.  The checks
    run outside the timed kv_swap calls."""
    from autx_workload import react, BASE_SEED, CONFIG_INDEX
    from paper_2502_13965_b200 import Scheduler, TraceDriver, SWAP_SM, SWAP_STAGED_DMA, SWAP_PER_CHUNK_MEMCPY
    L, chunk = 32, 32 << 10                 # LLaMA-3.1-8B: 32 layers x 8 KV heads x 128 x bf16 x 16 tok
    page = L * 2 * chunk                    # 2 MiB per logical block
    P, host_pages = 2560, 16384          # P >= the largest call's need (32768+4096 tokens)
    nblk = 2 * P                         # pool with room beyond the budget: swap-ins take blocks
                                         # freed by earlier steps, so both directions overlap
    kp = [torch.empty(nblk, chunk, dtype=torch.uint8, device="cuda") for _ in range(L)]
    vp = [torch.empty(nblk, chunk, dtype=torch.uint8, device="cuda") for _ in range(L)]
    host = torch.empty(host_pages * page, dtype=torch.uint8).pin_memory()
    lad = spec_ladder()
    results = {}

    def pat(cids, js, l, kv):  # one byte per (call, block, layer, K|V), the whole chunk
        return ((cids * 31 + js * 7 + l * 3 + kv) & 0xFF).to(torch.uint8)

    runs = (("sm", SWAP_SM, 1, 0), ("staged_dma", SWAP_STAGED_DMA, 1, 0),
            ("per_chunk_memcpy", SWAP_PER_CHUNK_MEMCPY, 1, 0),
            # the scheduler every 4 steps, 16 standby calls
            ("staged_dma_multistep_N4_X16", SWAP_STAGED_DMA, 4, 16))
    for name, mode, N, X in runs:
        tr = react(1000, seed=BASE_SEED + CONFIG_INDEX["react"])
        # the library and the engine's reads / writes of the pools on one stream (autx.h: all
        # device work is ordered on the context's stream)
        s = Scheduler(policy="plas", beta=(2, 1), max_batch=64, kv_budget=P, block_tokens=16,
                      max_calls=1 << 16, max_programs=1 << 14, n_gpu_blocks=nblk, max_blocks_per_call=P,
                      host_pages=host_pages, stream=torch.cuda.current_stream().cuda_stream,
                      sched_every=N, overprovision=X, **lad)
        d = TraceDriver(tr, s, log_lists=True)
        tot_b = tot_ms = 0.0
        b_d2h = b_h2d = 0
        n = 0
        t_at_peak = 0.0
        n_duplex = 0
        blocks_all = 0        # blocks swapped over every step of the run (both directions)
        written = {}          # call id -> leading blocks the engine has written
        checked = mismatched = 0
        for i in range(args.swap_steps + 20):
            if not d.skip_idle():
                break
            rec = d.step()
            st = s.kv_swap([x.data_ptr() for x in kp], [x.data_ptr() for x in vp], chunk,
                           host.data_ptr(), host.numel(), mode)
            blocks_all += rec["swap_out_blocks"] + rec["swap_in_blocks"]
            if i >= 20 and (st.bytes_d2h + st.bytes_h2d) > 0:
                tot_b += st.bytes_d2h + st.bytes_h2d
                tot_ms += st.ms
                b_d2h += st.bytes_d2h
                b_h2d += st.bytes_h2d
                t_at_peak += st.bytes_d2h / (link["d2h"] * 1e9) + st.bytes_h2d / (link["h2d"] * 1e9)
                n += 1
                n_duplex += int(st.duplex)
            # content check of the blocks that came back, then the engine's writes to new blocks
            offs, blks = s.block_table_host()
            ci, cj, cb, ni, nj, nb = [], [], [], [], [], []
            for k, cid in enumerate(rec["batch"]):
                mine = blks[offs[k]:offs[k + 1]]
                w = written.get(cid, 0)
                for j in range(len(mine)):
                    (ci if j < w else ni).append(cid)
                    (cj if j < w else nj).append(j)
                    (cb if j < w else nb).append(int(mine[j]))
                written[cid] = len(mine)
            admitted = set(rec["admit"])
            keep = [k for k in range(len(ci)) if ci[k] in admitted]  # only round trips need checking
            if keep:
                cids = torch.tensor([ci[k] for k in keep], device="cuda", dtype=torch.int64)
                js = torch.tensor([cj[k] for k in keep], device="cuda", dtype=torch.int64)
                idx = torch.tensor([cb[k] for k in keep], device="cuda", dtype=torch.int64)
                for l in range(L):
                    for kv, pools in ((0, kp), (1, vp)):
                        ok = (pools[l][idx] == pat(cids, js, l, kv)[:, None]).all(dim=1)
                        mismatched += int((~ok).sum())
                checked += len(keep) * L * 2
            if ni:
                cids = torch.tensor(ni, device="cuda", dtype=torch.int64)
                js = torch.tensor(nj, device="cuda", dtype=torch.int64)
                idx = torch.tensor(nb, device="cuda", dtype=torch.int64)
                for l in range(L):
                    for kv, pools in ((0, kp), (1, vp)):
                        pools[l][idx] = pat(cids, js, l, kv)[:, None].expand(-1, chunk)
        s.close()
        if n:
            gbs = tot_b / (tot_ms * 1e-3) / 1e9
            results[name] = {"GB/s": round(gbs, 2), "steps": n, "bytes_d2h": b_d2h, "bytes_h2d": b_h2d,
                             "ms_per_step": tot_ms / n, "frac_of_host_link": round(t_at_peak / (tot_ms * 1e-3), 4),
                             "frac_of_duplex_peak": round(gbs / link["duplex"], 4), "duplex_steps": n_duplex,
                             "sched_every": N, "overprovision": X,
                             "swapped_blocks_per_step": round(blocks_all / (i + 1), 2),
                             "content_check": {"chunks_checked": checked, "chunks_mismatched": mismatched,
                                               "ok": checked > 0 and mismatched == 0}}
    del kp, vp, host
    return results


# ------------------------------------------------------------------------------------------
# main arm
# ------------------------------------------------------------------------------------------
def main():
    args = parse()
    import torch
    rank, world, local = dist_init(args.gpus)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch.distributed as dist
    from paper_2502_13965_b200 import Scheduler, TraceDriver, ORDER_SELECT, ORDER_RADIX
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)   # one explicit stream for the library and the events
    torch.cuda.set_stream(stream)
    hbm_peak, peak_src = peaks()
    wl = dict(WORKLOADS[args.workload])
    active = args.active or wl["active"]
    if args.policy:
        wl["policy"] = args.policy

    t_gen = time.time()
    if world == 1:
        tr = make_trace(args.workload, active)
    else:
        # weak scaling: one shard per engine; every rank holds the whole (replicated) workload
        # because Alg. 2 routes each arrival to any engine
        from autx_workload.gen import concat
        tr = concat([make_trace(args.workload, active, 1000 * r) for r in range(world)],
                    name="%s_x%d" % (args.workload, world))
    t_gen = time.time() - t_gen
    lad = spec_ladder()
    beta = (1, 0) if args.beta == "inf" else (2, 1)
    gloo = os.environ.get("AUTX_DIST_BACKEND", "nccl") == "gloo"
    comm = None
    if world > 1 and not gloo:
        # the library's own NCCL communicator for autx_route (torch only ships the 128-byte id)
        from paper_2502_13965_b200.autx import comm_unique_id, comm_init
        box = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        comm = comm_init(box[0], rank, world, local)
    s = Scheduler(policy=wl["policy"], beta=beta, max_batch=wl["max_batch"], kv_budget=wl["kv_budget"],
                  block_tokens=16, max_calls=int(active * 1.25) + 4096, max_programs=tr.n_programs + 1024,
                  order_mode=ORDER_RADIX if args.order == "radix" else ORDER_SELECT,
                  device=local, stream=stream.cuda_stream, rank=rank, nranks=world, nccl_comm=comm, **lad)
    if world == 1:
        d = TraceDriver(tr, s, log_lists=False)
    else:
        from paper_2502_13965_b200.multi import MultiEngineDriver
        exchange = None                       # autx_route: record, ncclAllGather, apply, Alg. 2
        if gloo:
            nrec = s.route_record_bytes()

            def exchange(rec):
                parts = [torch.empty(nrec, dtype=torch.uint8) for _ in range(world)]
                torch.cuda.current_stream().synchronize()
                dist.all_gather(parts, rec.cpu())
                return torch.cat(parts).to(dev)

        def gather_ids(local_ids):
            out = [None] * world
            dist.all_gather_object(out, np.asarray(local_ids, np.int64))
            return out

        d = MultiEngineDriver(tr, s, rank, world, exchange, gather_ids,
                              lambda n: torch.zeros(n, dtype=torch.uint8, device=dev), log_lists=False)
    t_setup = time.time()
    d.step()                                  # step 0: registers the whole burst (setup)
    for _ in range(args.ff):
        d.step()
    t_setup = time.time() - t_setup

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    # ~1 ms spin while the host enqueues the step.  N > 1: none, because autx_route returns the
    # routes to the host (engine_out) mid-step, so the host waits on the device there anyway
    gate_cycles = 2_000_000 if world == 1 else 0

    def timed_step():
        d.prepare()                           # the workload model's host work, not the library's
        if not args.no_flush:
            flush.zero_()
        if gate_cycles:
            torch.cuda._sleep(gate_cycles)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        nc, na = d.issue()
        b.record(stream)
        rec = d.finish()
        b.synchronize()
        return a.elapsed_time(b), rec, nc, na

    s.set_timing(False)
    for _ in range(args.warmup):
        timed_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(os.path.join(ROOT, "gpurun_out", f"clocks_r{rank}.csv") if os.path.isdir(
        os.path.join(ROOT, "gpurun_out")) else f"/tmp/clocks_r{rank}.csv")
    clocks.start()
    from paper_2502_13965_b200.autx import kernel_launches
    ms, decisions, comps, arrs, promoted = [], 0, [], [], []
    launches0 = kernel_launches()
    for _ in range(args.steps):
        dt, rec, nc, na = timed_step()
        ms.append(dt)
        decisions += rec["n_active"]
        comps.append(nc)
        arrs.append(na)
        promoted.append(rec["n_promoted"])
    launches = kernel_launches() - launches0  # counted by the library at every launch
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ck = clocks.stop(local)
    st = s.step_stats()                       # selection shape of the last timed step
    # per-kernel device time: a separate pass with the library's CUDA events between the chain's
    # kernels (events serialise the PDL chain, so the parts add up to more than a step)
    s.set_timing(True)
    ev_ms = {"scan": [], "select+gather": [], "rank+finalize": []}
    for _ in range(30):
        timed_step()
        tm = s.last_step_timing()
        ev_ms["scan"].append(tm.scan_ms)
        ev_ms["select+gather"].append(tm.select_ms)
        ev_ms["rank+finalize"].append(tm.finalize_ms)
    # the undisturbed chain: %globaltimer stamps inside the kernels (no events), another pass
    s.set_timing(False, stamps=True)
    stamp_phase, stats = [], []
    for _ in range(30):
        timed_step()
        stamp_phase.append(s.phase_times().astype(np.int64))
        stats.append(s.step_stats())
    s.set_timing(False)
    spans = chain_spans(stamp_phase)
    # phases inside the finalize (raw stamps dbg[0, 32) of the step just run, thread 0 of the CTA,
    # us after the finalize's first stamp): [0, 10] the finalize body, [20, 25] its ordering
    # phases inside k_gather_ss (tile 0: selection known, positions known, records emitted) and
    # k_rank (CTA 0: keys in shared memory, compacted / split, ranked), us after each kernel's CTA 0
    # passed its PDL wait (dbg[57..59] and dbg[54..56], moved to [89..91] and [86..88] by finalize)
    sub_ph = {}
    for name, k, idx in (("gather", 3, (89, 90, 91)), ("rank", 4, (86, 87, 88))):
        vals = []
        for p in stamp_phase:
            b = int(p[64 + 3 * k])
            if b and all(int(p[i]) for i in idx):
                vals.append([int(p[i]) - b for i in idx])
        if vals:
            sub_ph[name] = [round(float(np.median([v[j] for v in vals])) / 1e3, 2) for j in range(3)]
    fin_ph = {}
    for i in list(range(0, 11)) + list(range(20, 26)):
        v = [int(p[i]) - int(p[0]) for p in stamp_phase if int(p[i]) and int(p[0])]
        if v:
            fin_ph[i] = round(float(np.median(v)) / 1e3, 2)
    total_ms = sum(ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dd = torch.tensor([decisions], device=dev, dtype=torch.float64)
        dist.all_reduce(dd)
        decisions = float(dd.item())
    value = decisions / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps

    # e2e: the same steps through the public API from the host, wall clock, no gate/flush
    e2e_dec, e2e_s, h2d, d2h, wall_s = 0, 0.0, 0, 0, 0.0
    split0 = dict(d.api_split)
    e2e_steps = min(args.steps, 200)
    # AUTX_E2E_FUSED=1: one boundary crossing per step (autx_step; one engine, no Eq. 2 parents).
    # Measured equal to the five-call sequence (50.7 vs 49.4 us per step): the host side is the
    # graph launch and the wait, not the crossings, so the default keeps the per-call split
    fused = world == 1 and wl["policy"] != "atlas_eq2" and bool(os.environ.get("AUTX_E2E_FUSED"))
    for _ in range(e2e_steps):
        nc = len(d.pending)
        api0 = d.api_s
        t0 = time.perf_counter()
        if fused:
            _, na, rec = d.run_fused()
        else:
            _, na = d.issue()
            rec = d.finish()
        wall_s += time.perf_counter() - t0
        e2e_s += d.api_s - api0
        e2e_dec += rec["n_active"]
        h2d += 8 * nc + 24 * na               # completion (slot, program row) + arrival records
        d2h += 8 * (rec["n_batch"] + rec["n_admit"] + rec["n_preempt"]) + 4 * rec["n_batch"] + 48
    n_compact, compact_us = s.compaction_stats()
    if world == 1:
        s.close()

    n_active = decisions / args.steps / world
    n_programs = st["n_programs"]
    algo_bytes = ALGO_BYTES_PER_CALL * n_active + ALGO_BYTES_PER_PROGRAM * n_programs
    design_bytes = DESIGN_BYTES_PER_ROW * st["n_rows"] + DESIGN_BYTES_PER_PROGRAM * n_programs
    achieved = algo_bytes / (ms_per_step * 1e-3) / 1e9
    ev_mean = {k: statistics.mean(v) for k, v in ev_ms.items()}
    span_k = {k: round(v[1] - v[0], 2) for k, v in (spans or {}).items()}
    dominant = max(span_k, key=span_k.get) if span_k else None
    traffic_bytes, traffic_src = ncu_traffic()
    if args.workload != "mcts" or args.order != "select" or wl["policy"] != "atlas" or args.beta != "2":
        traffic_bytes, traffic_src = None, "no ncu capture of this configuration"
    span_us = spans["finalize"][1] if spans and "finalize" in spans else None
    result = {
        "metric": "sched decisions/s at 1M active calls", "value": value, "unit": "decisions/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": wl["desc"] if world == 1 else
                   "%s x%d engines with Alg. 2 routing (BASELINE configs[4], weak)" % (args.workload, world),
                   "mean_active_calls_per_gpu": int(n_active), "table_rows": st["n_rows"],
                   "programs": n_programs, "policy": wl["policy"], "ladder": "SPEC K=8",
                   "beta": "inf" if args.beta == "inf" else "2",
                   "max_batch": wl["max_batch"], "kv_budget_blocks": wl["kv_budget"], "fast_forward_steps": args.ff,
                   "order": args.order, "l2": "flushed before every step (512 MiB write)" if not args.no_flush else "hot",
                   "parallelism": f"engines{world} (one scheduler per GPU)"},
        "gpu_launches": launches,
        "kernels_per_step": launches / args.steps,
        "roofline": {"bound": "hbm", "kernel": "the step (one graph launch of the PDL chain k_prologue -> "
                     "k_scan_tile -> k_gather_ss -> k_rank -> k_finalize)" if args.order == "select" else
                     "the step (prologue + k_keys + LSD passes + k_take + k_rank + k_finalize)",
                     "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4), "traffic": traffic_bytes, "traffic_source": traffic_src,
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": int(algo_bytes),
                     "algorithmic_bytes": "SURVEY 8(d): 52 B per active call + 16 B per program",
                     "timing": "CUDA events around each step's launch, L2 flushed before it (= ms_per_step)",
                     "dominant_kernel": dominant,
                     "dominant_by": "longest span inside the undisturbed chain (%globaltimer, CTA 0 past the PDL "
                                    "wait to the latest CTA end); see chain_us, kernel_event_ms and profiles/",
                     "design_bytes_per_launch": int(design_bytes),
                     "design_bytes": "13 B per table row (qf, prog, base, mtime) + 12 B per program row",
                     "chain_span_us": span_us,
                     "chain_span_source": "%globaltimer: the first kernel's CTA 0 to the finalize's end (30 steps, "
                                          "median); the rest of ms_per_step is launch and event overhead"},
        "step_ms": {"p10": float(np.percentile(ms, 10)), "p50": float(np.percentile(ms, 50)),
                    "p90": float(np.percentile(ms, 90)), "mean": statistics.mean(ms)},
        "chain_us": spans,
        "finalize_phases_us": fin_ph,
        "gather_rank_phases_us": sub_ph,
        "kernel_span_us": span_k,
        "kernel_event_ms": ev_mean,
        "state": {"promotions_per_step": statistics.mean(promoted),
                  "completions_per_step": statistics.mean(comps), "arrivals_per_step": statistics.mean(arrs),
                  "qstar": st["qstar"], "mprime": st["mprime"], "region_a": st["n_x"],
                  "region_b_mean": statistics.mean(x["n_b"] for x in stats),
                  "region_b_max": max(x["n_b"] for x in stats),
                  "queue_occupancy": st["queue_counts"][:lad["K"]],
                  "compactions": dict(count=n_compact, host_us_total=round(compact_us, 1), steps=d.t,
                                      note="G8 device compactions over the whole run (setup, fast-forward, "
                                           "warm-up, timed and e2e steps); their kernels run inside "
                                           "autx_register_call, so e2e includes them")},
        "e2e": {"value": e2e_dec / e2e_s, "unit": "decisions/s", "h2d_bytes_per_step": h2d // e2e_steps,
                "d2h_bytes_per_step": d2h // e2e_steps, "ms_per_step": e2e_s * 1e3 / e2e_steps,
                "timed": ("wall clock inside the C-ABI call autx_step (complete, end_program, register, "
                          "sched_step, step_wait in one crossing) + list copies" if fused else
                          "wall clock inside the C-ABI calls (complete, end_program, register, sched_step, "
                          "step_wait + list copies)") + " per step; H2D staging and D2H mirrors included",
                "api": "autx_step" if fused else "autx_complete/end_program/register_call/sched_step/step_wait",
                "harness_ms_per_step": (wall_s - e2e_s) * 1e3 / e2e_steps,
                "api_us_per_step": {k: round((v - split0.get(k, 0.0)) * 1e6 / e2e_steps, 1)
                                    for k, v in d.api_split.items()}},
        "setup_s": {"generate": round(t_gen, 1), "register_and_fast_forward": round(t_setup, 1)},
    }
    if ck:
        result["clocks"] = ck
    if rank == 0:
        print("sched:", json.dumps(result), file=sys.stderr, flush=True)
    if rank == 0 and world == 1 and not args.no_swap:
        link = host_link_peak(torch)
        try:
            sw = bench_swap(torch, args, link)
        except Exception as e:  # keep the sched line even if the swap phase fails
            sw = {"error": repr(e)}
        result["swap"] = {"host_link_peak_GBps": {k: round(v, 2) for k, v in link.items()},
                          "config": "react (BFCL-shaped) 1000 programs, PLAS, BS=64, P=2560 blocks, pool 5120 "
                                    "blocks, 8B geometry (32 layers x K|V x 32 KiB chunks = 2 MiB/block)",
                          "frac_of_host_link": "serial bound: d2h bytes / d2h peak + h2d bytes / h2d peak "
                                               "(> 1 only by overlapping the directions)",
                          "frac_of_duplex_peak": "GB/s over both directions / the measured two-stream "
                                                 "D2H + H2D copy peak", **sw}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, per_step, wall, _ = oracle_decisions_per_s(1_000_000, 2, 0)
        result["cpu_baseline"] = {"value": v, "unit": "decisions/s", "cores": 1, "kind": "oracle",
                                  "sample": f"the 1M-call burst of configs[3], 2 steps after the setup step, "
                                            f"{per_step:.2f} s/step single-threaded Python",
                                  "host_cores_available": os.cpu_count()}
    if rank == 0:
        line = json.dumps(result)
        print(line, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(line + "\n")
    if world > 1:
        s.close()
        if comm:
            from paper_2502_13965_b200.autx import comm_destroy
            comm_destroy(comm)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
