"""Multi-engine lockstep driver (BASELINE configs[4]): one scheduler per GPU,
one routing epoch per step.

Per step t on every rank (order of SURVEY §8(e); the oracle's simulate_multi follows it too):
  1. local completions of step t-1            -> autx_complete (rows freed, records built)
  2. epoch record (load after 1, records)      -> autx_route_pack into a device buffer
  3. all-gather of the G records               -> `exchange` (NCCL all_gather on GPUs, gloo in tests)
  4. every rank applies all G record sets to its replicated process table and routes the
     replicated arrival batch with Alg. 2     -> autx_route_apply (R22, R23)
  5. register the arrivals routed here, schedule -> autx_register_call, autx_sched_step
The workload side (DAG readiness) needs every rank's completed call ids, which `gather_ids`
all-gathers; it is harness state, not scheduler state.
"""
from __future__ import annotations

import time

import numpy as np

from .driver import TraceDriver


class MultiEngineDriver(TraceDriver):
    def __init__(self, trace, sched, rank, world, exchange, gather_ids, new_record, log_lists=True):
        super().__init__(trace, sched, log_lists=log_lists)
        self.rank, self.world = rank, world
        self.exchange = exchange          # record tensor -> gathered tensor (world records)
        self.gather_ids = gather_ids      # local np.int64 array -> list of arrays (all ranks)
        self.rec = new_record(sched.route_record_bytes())
        self.routes = []

    def issue(self):
        t = self.t
        s = self.s
        local = self.pending
        t0 = time.perf_counter()
        if len(local):
            s.complete(self.tr.call_id[local])
        s.route_pack(self.rec.data_ptr())
        gathered = self.exchange(self.rec)
        self.api_s += time.perf_counter() - t0
        all_done = np.sort(np.concatenate([np.asarray(x, np.int64) for x in self.gather_ids(local)]))
        ended = self._release(t, all_done)
        arr = self.arrivals(t)
        t0 = time.perf_counter()
        for pid in ended:
            s.end_program(pid)
        dest = s.route_apply(gathered.data_ptr(), arr)
        mine = arr[dest == self.rank]
        if len(mine):
            s.register(mine)
        s.sched_step(t, wait=False)
        self.api_s += time.perf_counter() - t0
        if self.log_lists:
            self.routes.append((t, [int(x) for x in arr["call_id"]], [int(x) for x in dest]))
        return len(local), len(mine)

    def run(self, max_steps=10 ** 9):
        # lockstep: every rank runs every step (no idle skipping: it needs global knowledge)
        for _ in range(max_steps):
            if self.finished():
                break
            self.step()
        return self.log
