"""Workload driver for the CUDA scheduler: feeds a synthetic trace through the C ABI step by
step.  It plays the roles the paper puts outside the scheduler: the agentic programs (DAG
readiness after parents finish plus interrupt delays), the frontend's
session start/end, and the model executor's decode lengths (hidden from the scheduler:
non-clairvoyance).  It holds none of the scheduling arithmetic.
"""
from __future__ import annotations

import time

import numpy as np

from .autx import CALL_DESC


class TraceDriver:
    def __init__(self, trace, sched, log_lists=True):
        self.tr = trace
        self.s = sched
        self.log_lists = log_lists
        C = trace.n_calls
        self.remaining = trace.decode.astype(np.int64).copy()
        self.n_par_left = np.diff(trace.par_ptr).astype(np.int64)
        # child adjacency (CSR) from the parent lists
        cnt = np.bincount(trace.par, minlength=C) if len(trace.par) else np.zeros(C, np.int64)
        self.cptr = np.concatenate([[0], np.cumsum(cnt)])
        owner = np.repeat(np.arange(C), np.diff(trace.par_ptr))
        self.child = owner[np.argsort(trace.par, kind="stable")]
        self.calls_left = np.diff(trace.first_call).astype(np.int64)
        self.ready = {}
        roots = np.nonzero(self.n_par_left == 0)[0]
        rt = trace.prog_arrival[trace.call_prog[roots]] + trace.delay[roots]
        for step in np.unique(rt):
            self.ready[int(step)] = list(roots[rt == step])
        self.pending = np.zeros(0, np.int64)   # call indices completed in the last step
        self.done = 0
        self.t = 0
        self.log = []
        self.total_wait = 0
        self.api_s = 0.0        # wall time spent inside the C ABI calls (the user-visible API)
        self.api_split = {}     # the same, per call

    def idx_of(self, cids):
        cids = np.asarray(cids, np.uint64)
        prog = (cids >> np.uint64(16)).astype(np.int64)
        return self.tr.first_call[prog] + (cids & np.uint64(0xFFFF)).astype(np.int64)

    def finished(self):
        return self.done == self.tr.n_calls

    def _release(self, t, done_idx):
        tr = self.tr
        ended = []
        for c in done_idx:
            self.done += 1
            p = tr.call_prog[c]
            self.calls_left[p] -= 1
            if self.calls_left[p] == 0:
                ended.append(int(tr.prog_id[p]))
            for ch in self.child[self.cptr[c]:self.cptr[c + 1]]:
                self.n_par_left[ch] -= 1
                if self.n_par_left[ch] == 0:
                    self.ready.setdefault(int(t + tr.delay[ch]), []).append(ch)
        return ended

    def arrivals(self, t):
        tr = self.tr
        cs = np.asarray(self.ready.pop(t, []), np.int64)
        d = np.zeros(len(cs), CALL_DESC)
        self.arr_idx = cs
        if len(cs) == 0:
            return d
        p = tr.call_prog[cs]
        d["call_id"] = tr.call_id[cs]
        d["program_id"] = tr.prog_id[p]
        d["arrival_step"] = t
        d["program_arrival_step"] = tr.prog_arrival[p]
        d["input_tokens"] = tr.input_tokens[cs]
        order = np.lexsort((d["call_id"], d["program_id"], d["program_arrival_step"]))
        self.arr_idx = cs[order]
        return d[order]

    def parents_csr(self, idx):
        """The arrivals' DAG parents as (offsets[n+1], parent call ids): the program tells the
        scheduler a call's parents when the call arrives."""
        tr = self.tr
        cnt = tr.par_ptr[idx + 1] - tr.par_ptr[idx]
        off = np.zeros(len(idx) + 1, np.int64)
        np.cumsum(cnt, out=off[1:])
        pos = np.repeat(tr.par_ptr[idx] - off[:-1], cnt) + np.arange(int(off[-1]))
        return off.astype(np.uint32), tr.call_id[tr.par[pos]]

    def prepare(self):
        """Workload side of the next step (no ABI call): the completed calls' ids, the programs
        they end, this step's arrivals.  Kept apart so a benchmark can do it before timing."""
        t = self.t
        ids = self.tr.call_id[self.pending]
        ended = self._release(t, self.pending)
        arr = self.arrivals(t)
        self._prepared = (t, ids, ended, arr)

    def issue(self):
        """Host half of one engine step: completions, session ends, arrivals, sched_step.
        Returns (n_completions, n_arrivals) without waiting for the device."""
        if getattr(self, "_prepared", None) is None or self._prepared[0] != self.t:
            self.prepare()
        t, ids, ended, arr = self._prepared
        self._prepared = None
        s = self.s
        nc = len(ids)
        pc = time.perf_counter
        t0 = pc()
        if nc:
            s.complete(ids)
        t1 = pc()
        for pid in ended:
            s.end_program(pid)
        t2 = pc()
        if len(arr):
            if getattr(s, "eq2", False):
                s.register_dag(arr, *self.parents_csr(self.arr_idx))
            else:
                s.register(arr)
        t3 = pc()
        s.sched_step(t, wait=False)
        t4 = pc()
        self.api_s += t4 - t0
        for k, dt in (("complete", t1 - t0), ("end_program", t2 - t1), ("register", t3 - t2), ("sched_step", t4 - t3)):
            self.api_split[k] = self.api_split.get(k, 0.0) + dt
        return nc, len(arr)

    def finish(self):
        """Waits for the step, logs it and runs the engine model (one decode step per batch
        call; calls whose hidden decode length is reached complete)."""
        s = self.s
        t0 = time.perf_counter()
        out = s.step_wait()
        t1 = time.perf_counter()
        batch, admit, preempt = s.lists()
        t2 = time.perf_counter()
        self.api_s += t2 - t0
        self.api_split["step_wait"] = self.api_split.get("step_wait", 0.0) + t1 - t0
        self.api_split["lists"] = self.api_split.get("lists", 0.0) + t2 - t1
        return self._record(out, batch, admit, preempt)

    def run_fused(self):
        """One engine step through the single-call entry point autx_step (completions, session
        ends, arrivals, sched_step, wait in one boundary crossing), then the lists.  Single
        engine, scalar ATLAS/PLAS/FCFS/MLFQ (EQ2 arrivals with parents use issue/finish)."""
        if getattr(self, "_prepared", None) is None or self._prepared[0] != self.t:
            self.prepare()
        t, ids, ended, arr = self._prepared
        self._prepared = None
        s = self.s
        pc = time.perf_counter
        t0 = pc()
        out = s.step(t, ids, ended, arr)
        t1 = pc()
        batch, admit, preempt = s.lists()
        t2 = pc()
        self.api_s += t2 - t0
        self.api_split["step"] = self.api_split.get("step", 0.0) + t1 - t0
        self.api_split["lists"] = self.api_split.get("lists", 0.0) + t2 - t1
        return len(ids), len(arr), self._record(out, batch, admit, preempt)

    def _record(self, out, batch, admit, preempt):
        s = self.s
        t = self.t
        rec = dict(t=t, n_batch=int(out.n_batch), swap_out_blocks=int(out.swap_out_blocks),
                   swap_in_blocks=int(out.swap_in_blocks), kv_blocks=int(out.kv_blocks),
                   n_active=int(out.n_active), n_promoted=int(out.n_promoted),
                   n_admit=int(out.n_admit), n_preempt=int(out.n_preempt))
        if self.log_lists:
            rec.update(batch=[int(x) for x in batch], admit=[int(x) for x in admit],
                       preempt=[int(x) for x in preempt])
            if getattr(out, "n_standby", 0):   # R32 over-provisioned resident calls
                rec["standby"] = [int(x) for x in s.standby()]
        self.log.append(rec)
        bi = self.idx_of(batch)
        self.remaining[bi] -= 1
        self.pending = bi[self.remaining[bi] == 0]
        self.t = t + 1
        return rec

    def skip_idle(self):
        """Jumps over steps with nothing active; returns False when the trace is done."""
        if self.finished():
            return False
        if len(self.pending) == 0 and self.s.num_active() == 0 and self.t not in self.ready:
            if not self.ready:
                return False
            self.t = min(self.ready)
        return True

    def step(self):
        """One engine step through the C ABI; returns the decision record."""
        self.issue()
        return self.finish()

    def run(self, max_steps=10 ** 9, fused=False):
        """Runs the trace; fused: one autx_step call per step instead of the five-call sequence."""
        for _ in range(max_steps):
            if not self.skip_idle():
                break
            if fused:
                self.run_fused()
            else:
                self.step()
        return self.log
