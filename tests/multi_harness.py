"""Helpers for the world_size-2 multi-engine tests (gloo).  `OracleSched` is a test-only
stand-in with the Scheduler's routing interface, backed by the CPU oracle, so the multi-engine
driver's host-side protocol (record exchange, replicated arrivals, lockstep readiness) can be
exercised on CPU; the GPU variant plugs in the real Scheduler."""
import ctypes
import os
import pickle
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REC_BYTES = 1 << 16


class OracleSched:
    def __init__(self, cfg, rank, world, router="locality"):
        from oracle.autellix import Engine, ProgramTable
        self.router, self.rr = router, {"next": 0}
        self.eng = Engine(cfg, table=ProgramTable(), check_formulations=False)
        self.cfg, self.rank, self.world = cfg, rank, world
        self.recs = []
        self.pins = {}
        self.t = 0
        self.last = None

    def route_record_bytes(self):
        return REC_BYTES

    def complete(self, ids):
        self.recs = self.eng.complete(self.t + 1 if self.last else 0, [int(x) for x in ids])

    def end_program(self, pid):
        self.ended = getattr(self, "ended", []) + [int(pid)]

    def route_pack(self, ptr):
        blob = pickle.dumps((self.eng.load(), self.recs))
        assert len(blob) + 8 <= REC_BYTES
        hdr = np.array([len(blob)], np.int64).tobytes()
        ctypes.memmove(ptr, hdr + blob, len(hdr) + len(blob))
        self.recs = []

    def route_apply(self, ptr, descs):
        from oracle.autellix import route, route_least_used, route_round_robin
        t = self.t + 1 if self.last else 0
        raw = ctypes.string_at(ptr, REC_BYTES * self.world)
        loads = []
        for r in range(self.world):
            chunk = raw[r * REC_BYTES:(r + 1) * REC_BYTES]
            n = int(np.frombuffer(chunk[:8], np.int64)[0])
            load, recs = pickle.loads(chunk[8:8 + n])
            loads.append(load)
            self.eng.apply_records(t, recs)
        for pid in getattr(self, "ended", []):
            self.eng.table.end_program(pid)
            self.pins.pop(pid, None)
        self.ended = []
        arr = [(int(d["call_id"]), int(d["program_id"]), int(d["input_tokens"])) for d in descs]
        for _, pid, _ in arr:       # replicated process table: every rank creates every entry
            self.eng.table.ensure(pid, t)
        if self.router == "least_used":
            return np.array(route_least_used(arr, loads), np.int32)
        if self.router == "round_robin":
            return np.array(route_round_robin(arr, self.world, self.rr), np.int32)
        return np.array(route(arr, loads, self.pins, self.cfg.token_threshold), np.int32)

    def register(self, descs):
        t = int(descs["arrival_step"][0])
        self.eng.register(t, [(int(d["call_id"]), int(d["program_id"]), int(d["arrival_step"]),
                               int(d["program_arrival_step"]), int(d["input_tokens"])) for d in descs])

    def sched_step(self, t, wait=True):
        self.t = t
        self.eng.demote_and_promote()
        self.last = self.eng.schedule(t)

    def step_wait(self):
        class O:
            pass
        o = O()
        r = self.last
        o.n_batch, o.n_admit, o.n_preempt = len(r["batch"]), len(r["admit"]), len(r["preempt"])
        o.swap_out_blocks, o.swap_in_blocks = r["swap_out"], r["swap_in"]
        o.kv_blocks, o.n_active, o.n_promoted = r["kv_blocks"], r["n_active"], 0
        return o

    def lists(self):
        r = self.last
        return tuple(np.array(r[k], np.uint64) for k in ("batch", "admit", "preempt"))

    def num_active(self):
        return len(self.eng.calls)


def run_rank(rank, world, port, out_path, use_gpu, trace_name, seed, cfg_kw, router="locality"):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.autellix import Config
    from paper_2502_13965_b200.multi import MultiEngineDriver
    tr = make_trace(trace_name, seed)
    cfg = Config(**cfg_kw)
    if use_gpu == "nccl":
        # autx_route: the library's own NCCL communicator, one GPU per rank
        from paper_2502_13965_b200 import Scheduler
        from paper_2502_13965_b200.autx import comm_unique_id, comm_init
        torch.cuda.set_device(rank)
        box = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        comm = comm_init(box[0], rank, world, rank)
        s = Scheduler(policy=cfg.policy, K=cfg.K, q_hi=cfg.q_hi, quanta=cfg.quanta, beta=cfg.beta,
                      max_batch=cfg.max_batch, kv_budget=cfg.kv_budget, block_tokens=cfg.block_tokens,
                      max_calls=1 << 15, max_programs=1 << 12, token_threshold=cfg.token_threshold,
                      device=rank, rank=rank, nranks=world, route_policy=router, nccl_comm=comm)
        new_record, exchange = None, None
    elif use_gpu:
        from paper_2502_13965_b200 import Scheduler
        torch.cuda.set_device(0)
        s = Scheduler(policy=cfg.policy, K=cfg.K, q_hi=cfg.q_hi, quanta=cfg.quanta, beta=cfg.beta,
                      max_batch=cfg.max_batch, kv_budget=cfg.kv_budget, block_tokens=cfg.block_tokens,
                      max_calls=1 << 15, max_programs=1 << 12, token_threshold=cfg.token_threshold,
                      rank=rank, nranks=world, route_policy=router)

        def new_record(nbytes):
            return torch.zeros(nbytes, dtype=torch.uint8, device="cuda")

        def exchange(rec):
            torch.cuda.synchronize()
            parts = [torch.zeros_like(rec).cpu() for _ in range(world)]
            dist.all_gather(parts, rec.cpu())
            return torch.cat(parts).cuda()
    else:
        s = OracleSched(cfg, rank, world, router)

        def new_record(nbytes):
            return torch.zeros(nbytes, dtype=torch.uint8)

        def exchange(rec):
            parts = [torch.zeros_like(rec) for _ in range(world)]
            dist.all_gather(parts, rec)
            return torch.cat(parts).contiguous()

    def gather_ids(local):
        out = [None] * world
        dist.all_gather_object(out, np.asarray(local, np.int64))
        return out

    d = MultiEngineDriver(tr, s, rank, world, exchange, gather_ids, new_record)
    log = d.run(max_steps=100000)
    if use_gpu == "nccl":
        from paper_2502_13965_b200.autx import comm_destroy
        s.close()
        comm_destroy(comm)
    recs = [(r["t"], r["batch"], r["admit"], r["preempt"]) for r in log if r["batch"] or r["preempt"]]
    with open(out_path, "wb") as f:
        pickle.dump({"log": recs, "routes": d.routes}, f)
    dist.barrier()
    dist.destroy_process_group()


def run_world(tmp_path, use_gpu, trace_name, seed, cfg_kw, world=2, router="locality"):
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    outs = [str(tmp_path / f"rank{r}.pkl") for r in range(world)]
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=run_rank, args=(r, world, port, outs[r], use_gpu, trace_name, seed, cfg_kw, router))
          for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(600)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    return [pickle.load(open(o, "rb")) for o in outs]


def make_trace(trace_name, seed):
    """The multi-engine tests' traces; "golden_route": tests/golden/route_2engine.json."""
    from autx_workload import random_tiny, chatbot, mcts_mapreduce
    if trace_name == "golden_route":
        from test_oracle_route_golden import golden_trace_and_config
        return golden_trace_and_config()[1]
    return {"tiny": lambda: random_tiny(seed, max_programs=6), "chatbot": lambda: chatbot(60),
            "mcts": lambda: mcts_mapreduce(8)}[trace_name]()


def golden_route():
    """(config kwargs, expected routes, expected per-engine records) of the golden trace."""
    import json
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "route_2engine.json")))
    c = g["config"]
    cfg = dict(policy=c["policy"], K=c["K"], q_hi=tuple(c["q_hi"]), quanta=tuple(c["quanta"]), beta=tuple(c["beta"]),
               max_batch=c["max_batch"], token_threshold=c["token_threshold"])
    routes = [(t, list(cids), list(dest)) for t, cids, dest in g["routes"]]
    logs = [[(t, b, a, p) for t, b, a, p in eng] for eng in g["batches"]]
    return cfg, routes, logs


def oracle_multi(trace_name, seed, cfg_kw, world=2, router="locality"):
    from oracle.autellix import Config, simulate_multi
    tr = make_trace(trace_name, seed)
    logs, routes = simulate_multi(tr, Config(**cfg_kw), world, router=router)
    out = [[(r["t"], r["batch"], r["admit"], r["preempt"]) for r in lg if r["batch"] or r["preempt"]]
           for lg in logs]
    return out, [(t, c, d) for t, c, d in routes]
