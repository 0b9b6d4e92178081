"""Program-level metrics and the clairvoyant SRPT bound.

TEST INFRASTRUCTURE ONLY, like the rest of `oracle/`: only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s reference / cpu_baseline legs may import it; the product path never does.

Written from PAPER.md §6.2 "Metrics" and footnote 2, and §6.5.3
"Comparison to Optimal Scheduling", in the engine-step time unit (reading R17):

* program-level token latency = program response time / tokens generated; for a
  multi-threaded program the response time is the critical path's (footnote 2);
* response time excludes interrupt delays (tool calls, human turns), which are "unrelated to LLM
  serving" (reading R33): the realized critical path is walked back from the
  program's last completion through, at each call, the parent that completed last, and the
  interrupt delays of the calls on it are subtracted;
* tokens = one per decode step of every call of the program (the idealized engine emits one token
  per call per step);
* SRPT, the clairvoyant comparison policy of §6.5.3: "exposing each program's total LLM calls and
  decode steps a priori", priority = the program's remaining decode steps over all its
  unfinished calls, ties by program arrival, program id, call registration;
  scheduling-only ("each continuous-batching step is identical"): BS calls per step,
  preemptive every step, no KV budget.

Every metric is computed from a decision log (the batch of every step) and the trace, so the
CUDA path's logs are scored by the same code as the oracle's.
"""
from __future__ import annotations

import numpy as np

from .autellix import Workload


def completion_steps(trace, log):
    """Step at which each call's completion is processed (the step after its last decode step;
    reading R29), from a log of per-step records with 't' and 'batch' (call ids)."""
    index = {int(cid): i for i, cid in enumerate(trace.call_id)}
    last = np.full(trace.n_calls, -1, np.int64)
    for rec in log:
        for cid in rec["batch"]:
            last[index[int(cid)]] = rec["t"]
    assert np.all(last >= 0), "every call must have run"
    return last + 1


def program_latency(trace, log):
    """Per program: (response steps, tokens, token latency), P:L350-354 and footnote 2 (R33)."""
    done = completion_steps(trace, log)
    out = []
    for p in range(trace.n_programs):
        a, b = int(trace.first_call[p]), int(trace.first_call[p + 1])
        calls = range(a, b)
        end = max(calls, key=lambda c: (done[c], c))          # the program's last completion
        finish = int(done[end])
        # realized critical path: back through the parent that completed last, summing the
        # interrupt delays of the calls on it (they are not serving time)
        delays, c = 0, end
        while True:
            delays += int(trace.delay[c])
            ps = [int(x) for x in trace.parents(c)]
            if not ps:
                break
            c = max(ps, key=lambda k: (done[k], k))
        response = finish - int(trace.prog_arrival[p]) - delays
        tokens = int(trace.decode[a:b].sum())
        out.append((response, tokens, response / tokens))
    return out


def latency_summary(lat):
    """Mean, P95 and P99 of the program-level token latency (Fig. 12 / Fig. 13)."""
    x = np.array([v for _, _, v in lat], dtype=np.float64)
    return dict(mean=float(x.mean()), p95=float(np.percentile(x, 95)), p99=float(np.percentile(x, 99)),
                programs=len(x))


def simulate_srpt(trace, max_batch, max_steps=1_000_000):
    """The clairvoyant SRPT scheduler of §6.5.3 over a whole trace; returns the log (records
    with 't', 'batch')."""
    wl = Workload(trace)
    remaining_prog = np.array([int(trace.decode[trace.first_call[p]:trace.first_call[p + 1]].sum())
                               for p in range(trace.n_programs)], np.int64)
    index = {int(cid): i for i, cid in enumerate(trace.call_id)}
    active = {}   # call index -> registration sequence
    seq = 0
    log = []
    completed = []
    for t in range(max_steps):
        if wl.finished():
            break
        wl.release(t, completed)
        for a in wl.arrivals(t):
            active[index[a[0]]] = seq
            seq += 1

        def key(c):
            p = int(trace.call_prog[c])
            return (int(remaining_prog[p]), int(trace.prog_arrival[p]), int(trace.prog_id[p]), active[c])

        batch = [int(trace.call_id[c]) for c in sorted(active, key=key)[:max_batch]]
        log.append(dict(t=t, batch=batch))
        completed = wl.ran(t, batch)
        for cid in batch:
            remaining_prog[int(trace.call_prog[index[cid]])] -= 1
        for c in completed:
            del active[c]
    assert wl.finished(), "SRPT simulation did not finish"
    return log


def makespan(trace, log):
    """Offline makespan (§6.5.1, "makespan of all programs"; Fig. 9): steps from
    the first program arrival to the last call completion (completion = the step after its last
    decode step, reading R29)."""
    return int(completion_steps(trace, log).max()) - int(np.min(trace.prog_arrival))


def total_wait(trace, log):
    """Steps every call spent active but not running (the Fig. 2 metric, reading R16)."""
    done = completion_steps(trace, log)
    ran = np.zeros(trace.n_calls, np.int64)
    index = {int(cid): i for i, cid in enumerate(trace.call_id)}
    for rec in log:
        for cid in rec["batch"]:
            ran[index[int(cid)]] += 1
    # a call is active from its arrival (parents done + delay) to its completion
    arrive = np.zeros(trace.n_calls, np.int64)
    for c in range(trace.n_calls):
        ps = trace.parents(c)
        start = max((int(done[k]) for k in ps), default=int(trace.prog_arrival[trace.call_prog[c]]))
        arrive[c] = start + int(trace.delay[c])
    return int(((done - arrive) - ran).sum())


def sweep(make_trace, rates, policies, max_batch, seeds=(0,)):
    """Mean / P95 / P99 program token latency per (arrival rate, policy) (a
    directional Fig. 12 / Fig. 18 reproduction).  policies: name -> callable(trace) -> log."""
    rows = []
    for lam in rates:
        for name, run in policies.items():
            acc = []
            for s in seeds:
                tr = make_trace(lam, s)
                acc.append(latency_summary(program_latency(tr, run(tr))))
            rows.append(dict(rate=lam, policy=name, **{k: float(np.mean([a[k] for a in acc]))
                                                       for k in ("mean", "p95", "p99")}))
    return rows
