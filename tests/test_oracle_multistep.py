"""Oracle pins for multi-step scheduling with over-provisioning (
reading R32 in DESIGN.md).

  * tests/golden/multistep.json: two hand-derived traces (a standby call filling a slot freed
    mid-window; a demotion deferred to the next scheduling point), every list of every step;
  * reductions: N = 1 gives the plain path's batches for any X (the resident set's first BS
    calls are the plain prefix), and N = 1, X = 0 is the plain path record for record;
  * invariants over random traces x N x X x KV budgets: batch <= BS, standby <= X, the resident
    set fits P, admit / preempt are the set differences with the previous resident set, the
    scheduler runs at least every N steps and ordering-dependent changes (admissions of calls
    that were not resident) happen only at scheduling points, swap bytes follow the ledger;
    every call completes.
"""
import json
import os

import pytest

from autx_workload.gen import dag_trace, random_tiny
from oracle.autellix import Config, Engine, Workload, simulate, ceil_div, FCFS, MLFQ, PLAS, ATLAS
from oracle.metrics import total_wait

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "multistep.json")))


def golden_trace(case):
    progs = [dict(decode=p["decode"], parents=[[]] * len(p["decode"])) for p in case["programs"]]
    return dag_trace(case["name"], progs, [p["arrival"] for p in case["programs"]])


@pytest.mark.parametrize("case", G["cases"], ids=[c["name"] for c in G["cases"]])
def test_golden_multistep(case):
    tr = golden_trace(case)
    c = dict(case["config"])
    c["q_hi"], c["quanta"] = tuple(c["q_hi"]), tuple(c["quanta"])
    log, m = simulate(tr, Config(**c).check())
    prog = lambda cids: [int(x) >> 16 for x in cids]   # one call per program: program index
    got = [dict(t=r["t"], batch=prog(r["batch"]), standby=prog(r.get("standby", [])),
                admit=prog(r["admit"]), preempt=prog(r["preempt"])) for r in log]
    n = len(case["steps"])
    assert got[:n] == case["steps"]
    assert all(not r["batch"] for r in got[n:])      # the last completions' bookkeeping step
    assert m["total_wait"] == case["total_wait"] == total_wait(tr, log)


LADDERS = [dict(K=1, q_hi=(), quanta=(None,)), dict(K=2, q_hi=(1,), quanta=(1, None)),
           dict(K=3, q_hi=(2, 5), quanta=(1, 2, None))]


def cfg(i, policy, N, X):
    return Config(policy=policy, max_batch=1 + i % 3, kv_budget=(None, 10, 16)[(i // 3) % 3],
                  beta=((1, 0), (2, 1))[(i // 9) % 2], block_tokens=4, block_bytes=64,
                  sched_every=N, overprovision=X, **LADDERS[i % 3]).check()


class CheckedEngine(Engine):
    """Engine.step's dispatch (scheduling point or window step) with the step invariants."""

    def step(self, t, completed, arrivals, parents=None):
        prev_res = self.prev_batch + self.standby
        self.apply_records(t, self.complete(t, completed))
        self.register(t, arrivals, parents)
        carried = self.prev_batch + self.standby
        sched, since = self.sched_point(), self.since
        if sched:
            self.demote_and_promote()
        kvb = {x: ceil_div(c.input_tokens + c.exec + 1, self.cfg.block_tokens) for x, c in self.calls.items()}
        held = {x: (c.held, c.exec) for x, c in self.calls.items()}
        resident_before = {x for x, c in self.calls.items() if c.resident}
        rec = self.schedule(t) if sched else self.window(t)
        self.since = 1 if sched else self.since + 1
        BS, X, P, N = self.cfg.max_batch, self.cfg.overprovision, self.cfg.kv_budget, self.cfg.sched_every
        standby = rec.get("standby", [])
        res = rec["batch"] + standby
        assert len(rec["batch"]) <= BS and len(standby) <= X
        assert not standby or len(rec["batch"]) == BS
        assert P is None or sum(kvb[x] for x in res) <= P
        assert (len(rec["batch"]) > 0) == (len(self.calls) > 0)
        assert rec["admit"] == [x for x in res if x not in resident_before]
        assert rec["preempt"] == [x for x in prev_res if x in self.calls and x not in set(res)]
        assert rec["swap_out"] == 64 * sum(held[x][0] for x in rec["preempt"] if held[x][1] > 0)
        assert rec["swap_in"] == 64 * sum(held[x][0] for x in rec["admit"] if held[x][1] > 0)
        if not sched:
            assert since < N and carried
            assert rec["admit"] == []                     # window: only resident calls run
            assert res == carried[:len(res)]              # carried order, cut at the first misfit
        return rec


def run_checked(tr, c):
    eng = CheckedEngine(c)
    wl = Workload(tr)
    completed, log, gap = [], [], 0
    for t in range(20_000):
        if wl.finished():
            break
        cids = [int(tr.call_id[x]) for x in completed]
        ended = wl.release(t, completed)
        arr = wl.arrivals(t)
        rec = eng.step(t, cids, arr)
        gap = gap + 1 if eng.since != 1 else 0
        assert gap < c.sched_every                        # the scheduler runs at least every N steps
        for pid in ended:
            eng.end_program(pid)
        log.append(rec)
        completed = wl.ran(t, rec["batch"])
    assert wl.finished()
    return log


@pytest.mark.parametrize("seed", range(120))
def test_random_multistep_invariants(seed):
    tr = random_tiny(seed, max_programs=5)
    for k, (policy, N, X) in enumerate([(PLAS, 2, 1), (ATLAS, 3, 2), (MLFQ, 2, 0), (FCFS, 4, 1)]):
        try:
            run_checked(tr, cfg(seed * 4 + k, policy, N, X))
        except ValueError as e:   # initial kvb > P (R13) or growth past P (R14)
            assert "exceeds" in str(e)


@pytest.mark.parametrize("seed", range(80))
def test_n1_gives_the_plain_batches_for_any_x(seed):
    """With the scheduler every step, the resident set's first BS calls are the plain cutoff's
    prefix (both walks stop at the same misfit), so the batch sequence cannot depend on X."""
    tr = random_tiny(seed, max_programs=5)
    for policy in (PLAS, ATLAS):
        base = cfg(seed, policy, 1, 0)
        try:
            plain = simulate(tr, base)[0]
        except ValueError:
            continue
        for X in (1, 3):
            c = cfg(seed, policy, 1, X)
            assert [r["batch"] for r in simulate(tr, c)[0]] == [r["batch"] for r in plain]


@pytest.mark.parametrize("seed", range(40))
def test_n1_x0_is_the_plain_path(seed):
    tr = random_tiny(seed)
    c = cfg(seed, ATLAS, 1, 0)
    plain = Config(**{k: v for k, v in c.__dict__.items() if k not in ("sched_every", "overprovision")})
    try:
        a = simulate(tr, plain)[0]
    except ValueError:
        return
    assert simulate(tr, c)[0] == a


def test_overprovisioning_cuts_swaps_on_a_react_shaped_trace():
    """Directional check of the paper's claim ("reduces total swaps"): on a small
    BFCL/ReAct-shaped trace with a binding KV budget, N = 4 with X = BS/4 swaps fewer blocks than
    the plain every-step scheduler."""
    from autx_workload import react
    tr = react(300, seed=11)
    base = dict(policy=PLAS, K=8, q_hi=(2, 8, 32, 128, 512, 2048, 8192),
                quanta=(2, 6, 24, 96, 384, 1536, 6144, None), beta=(2, 1), max_batch=16,
                kv_budget=2560, block_tokens=16, block_bytes=1)
    plain = simulate(tr, Config(**base).check(), check_formulations=False)[0]
    multi = simulate(tr, Config(**base, sched_every=4, overprovision=4).check(), check_formulations=False)[0]
    swaps = lambda log: sum(r["swap_out"] + r["swap_in"] for r in log)
    assert swaps(multi) < 0.6 * swaps(plain)     # measured: 415,164 vs 894,866 blocks
