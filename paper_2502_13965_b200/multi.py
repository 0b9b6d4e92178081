"""Multi-engine lockstep driver (BASELINE configs[4]): one scheduler per GPU,
one routing epoch per step.

Per step t on every rank (order of SURVEY §8(e); the oracle's simulate_multi follows it too):
  1. local completions of step t-1            -> autx_complete (rows freed, records built)
  2. epoch record (load after 1, records), all-gather of the G records, apply all G record sets
     to the replicated process table (R22), route the replicated arrival batch with Alg. 2 (R23)
                                               -> autx_route: one collective (ncclAllGather on the
                                                  library's communicator), or, with an
                                                  `exchange` callable (gloo tests), the split
                                                  autx_route_pack / exchange / autx_route_apply
  3. register the arrivals routed here, schedule -> autx_register_call, autx_sched_step
The workload side (DAG readiness) needs every rank's completed call ids, which `gather_ids`
all-gathers in `prepare()`; it is harness state (the meta-engine's), not scheduler state,
so a benchmark does it before its timed region.
"""
from __future__ import annotations

import time

import numpy as np

from .driver import TraceDriver


class MultiEngineDriver(TraceDriver):
    def __init__(self, trace, sched, rank, world, exchange, gather_ids, new_record, log_lists=True):
        super().__init__(trace, sched, log_lists=log_lists)
        self.rank, self.world = rank, world
        self.exchange = exchange          # None: autx_route (in-library NCCL); else record -> gathered
        self.gather_ids = gather_ids      # local np.int64 array -> list of arrays (all ranks)
        self.rec = new_record(sched.route_record_bytes()) if exchange is not None else None
        self.routes = []

    def prepare(self):
        """Harness side of step t (no ABI call): every engine's completed calls (for DAG
        readiness), the programs they end, the replicated arrival batch."""
        t = self.t
        local = self.pending
        all_done = np.sort(np.concatenate([np.asarray(x, np.int64) for x in self.gather_ids(local)]))
        ended = self._release(t, all_done)
        self._prepared = (t, self.tr.call_id[local], ended, self.arrivals(t))

    def issue(self):
        if getattr(self, "_prepared", None) is None or self._prepared[0] != self.t:
            self.prepare()
        t, ids, ended, arr = self._prepared
        self._prepared = None
        s = self.s
        t0 = time.perf_counter()
        if len(ids):
            s.complete(ids)
        if self.exchange is None:
            for pid in ended:
                s.end_program(pid)
            dest = s.route(arr)
        else:
            s.route_pack(self.rec.data_ptr())
            gathered = self.exchange(self.rec)
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
        return len(ids), len(mine)

    def run(self, max_steps=10 ** 9):
        # lockstep: every rank runs every step (no idle skipping: it needs global knowledge)
        for _ in range(max_steps):
            if self.finished():
                break
            self.step()
        return self.log
