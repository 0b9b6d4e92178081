"""Oracle pins: invariants, reductions and brute force over random tiny traces
(SURVEY.md §8(c))."""
import copy
import itertools

import numpy as np
import pytest

from autx_workload import random_tiny, fig2
from oracle.autellix import (Engine, Config, simulate, simulate_multi, PLAS, ATLAS, MLFQ, FCFS,
                             ATLAS_EQ2, Workload, ceil_div)

LADDERS = [
    dict(K=1, q_hi=(), quanta=(None,)),
    dict(K=2, q_hi=(1,), quanta=(1, None)),
    dict(K=3, q_hi=(2, 5), quanta=(1, 2, None)),
    dict(K=4, q_hi=(1, 3, 6), quanta=(2, 1, 3, 2)),
]
BETAS = [(1, 0), (2, 1), (1, 2), (5, 3)]
BUDGETS = [None, 8, 12]


def cfg_for(i, policy):
    lad = LADDERS[i % len(LADDERS)]
    return Config(policy=policy, max_batch=1 + i % 3, kv_budget=BUDGETS[(i // 3) % 3],
                  beta=BETAS[(i // 9) % 4], block_tokens=4, block_bytes=64, **lad)


class CheckedEngine(Engine):
    """Engine that asserts the step invariants while it runs."""

    def demote_and_promote(self):
        super().demote_and_promote()
        num, den = self.cfg.beta
        for c in self.calls.values():
            assert c.quanta is None or c.quanta >= 1
            if den:
                W = self.table.pwait[c.pid] + c.wait
                T = self.table.svc[c.pid] + c.mtime
                # after the scan every call is below the threshold or was just promoted
                assert (W * den < num * T) or (W == 0 and T == 0) or (c.wait == 0 and c.mtime == 0)

    def schedule(self, t):
        before = copy.deepcopy(self.calls)
        prev = list(self.prev_batch)
        rec = super().schedule(t)
        batch = rec["batch"]
        BS, P = self.cfg.max_batch, self.cfg.kv_budget
        kvb = {cid: ceil_div(c.input_tokens + c.exec + 1, self.cfg.block_tokens) for cid, c in before.items()}
        # capacity
        assert len(batch) <= BS and (P is None or sum(kvb[x] for x in batch) <= P)
        # work conservation in prefix form: non-empty batch whenever a call is active
        assert (len(batch) > 0) == (len(before) > 0)
        # brute force: the batch is the longest feasible prefix of the key order
        order = sorted(before.values(), key=lambda c: (c.q, c.arr, 0 if c.running else 1, c.seq))
        best = 0
        for n in range(len(order) + 1):
            pre = order[:n]
            if len(pre) <= BS and (P is None or sum(kvb[c.cid] for c in pre) <= P):
                best = n
            else:
                break
        assert batch == [c.cid for c in order[:best]]
        # priority semantics: no batch call has a larger key than a waiting call that fits
        # (prefix form: the first excluded call does not fit)
        if best < len(order):
            nxt = order[best]
            assert best + 1 > BS or (P is not None and sum(kvb[x] for x in batch) + kvb[nxt.cid] > P)
        # admit / preempt are the set differences with the resident set
        resident = [x for x in prev]
        assert rec["admit"] == [x for x in batch if x not in resident]
        assert rec["preempt"] == [x for x in resident if x not in batch]
        return rec


def run_checked(tr, cfg):
    eng = CheckedEngine(cfg)
    wl = Workload(tr)
    completed, log = [], []
    svc_hist = {}
    for t in range(10_000):
        if wl.finished():
            break
        cids = [int(tr.call_id[c]) for c in completed]
        ended = wl.release(t, completed)
        arr = wl.arrivals(t)
        rec = eng.step(t, cids, arr, wl.parents_of(arr) if cfg.policy == ATLAS_EQ2 else None)
        for pid, s in eng.table.svc.items():
            assert s >= svc_hist.get(pid, 0)       # monotone table
            svc_hist[pid] = s
        for pid in ended:
            eng.end_program(pid)
        log.append(rec)
        completed = wl.ran(t, rec["batch"])
    assert wl.finished()
    return log


@pytest.mark.parametrize("seed", range(300))
def test_random_tiny_invariants(seed):
    tr = random_tiny(seed)
    for p, policy in enumerate((FCFS, MLFQ, PLAS, ATLAS)):
        cfg = cfg_for(seed * 4 + p, policy)
        try:
            run_checked(tr, cfg)
        except ValueError as e:
            assert "exceeds the KV budget" in str(e)


@pytest.mark.parametrize("seed", range(150))
def test_random_tiny_invariants_eq2(seed):
    """The step invariants under exact Eq. 2 inheritance (R31), DAG traces with forks and joins."""
    tr = random_tiny(seed, max_calls=6)
    try:
        run_checked(tr, cfg_for(seed * 4 + 3, ATLAS_EQ2))
    except ValueError as e:  # initial kvb > P (R13) or a call outgrowing P while it decodes (R14, R30)
        assert "exceeds the KV budget" in str(e) or "exceeds the budget" in str(e)


@pytest.mark.parametrize("seed", range(50))
def test_determinism(seed):
    tr = random_tiny(seed)
    cfg = cfg_for(seed, ATLAS)
    cfg.kv_budget = None
    a = simulate(tr, cfg)[0]
    b = simulate(random_tiny(seed), cfg)[0]
    assert a == b


@pytest.mark.parametrize("seed", range(100))
def test_plas_k1_equals_fcfs_on_one_call_programs(seed):
    """S:L354 reduction: PLAS(K=1, infinite quantum) on one-call programs == FCFS."""
    tr = random_tiny(seed, max_calls=1, max_programs=6)
    f = simulate(tr, Config(policy=FCFS, K=1, q_hi=(), quanta=(None,), max_batch=2))[0]
    p = simulate(tr, Config(policy=PLAS, K=1, q_hi=(), quanta=(None,), max_batch=2))[0]
    assert [r["batch"] for r in f] == [r["batch"] for r in p]


@pytest.mark.parametrize("seed", range(100))
def test_atlas_equals_plas_on_chains(seed):
    """S:L355 reduction: ATLAS == PLAS on chain-only workloads."""
    tr = random_tiny(seed, dag=False)
    for lad in LADDERS[1:]:
        a = simulate(tr, Config(policy=ATLAS, max_batch=2, **lad))[0]
        b = simulate(tr, Config(policy=PLAS, max_batch=2, **lad))[0]
        assert [r["batch"] for r in a] == [r["batch"] for r in b]


@pytest.mark.parametrize("seed", range(40))
def test_fcfs_one_call_closed_form(seed):
    """FCFS, one call per program, BS=1, all at t=0, no KV limit: calls run back to back
    in program order; total wait = sum over calls of the decode steps of those before."""
    tr = random_tiny(seed, max_calls=1, max_programs=6, max_arrival=0)
    log, m = simulate(tr, Config(policy=FCFS, K=1, q_hi=(), quanta=(None,), max_batch=1))
    d = [int(x) for x in tr.decode]
    assert m["total_wait"] == sum(sum(d[:i]) for i in range(len(d)))


@pytest.mark.parametrize("seed", range(40))
def test_multi_engine_g1_equals_single(seed):
    tr = random_tiny(seed)
    cfg = cfg_for(seed, ATLAS)
    cfg.kv_budget = None
    single = simulate(tr, cfg, check_formulations=False)[0]
    logs, routes = simulate_multi(tr, cfg, 1)
    assert [r["batch"] for r in logs[0]] == [r["batch"] for r in single]
    assert all(all(d == 0 for d in r[2]) for r in routes)


@pytest.mark.parametrize("seed", range(40))
def test_multi_engine_invariants(seed):
    """Lockstep G=3: every call is routed exactly once and runs only on its engine;
    replicated table monotone; each engine's batch <= BS."""
    tr = random_tiny(seed, max_programs=6)
    cfg = cfg_for(seed, PLAS)
    cfg.kv_budget = None
    cfg.token_threshold = 8
    logs, routes = simulate_multi(tr, cfg, 3)
    where = {}
    for t, cids, dest in routes:
        for c, d in zip(cids, dest):
            assert c not in where
            where[c] = d
    assert len(where) == tr.n_calls
    for e, log in enumerate(logs):
        for r in log:
            assert len(r["batch"]) <= cfg.max_batch
            assert all(where[c] == e for c in r["batch"])


def test_starvation_bound_finite_beta():
    """with finite beta a waiting call is eventually promoted to Q1."""
    e = Engine(Config(policy=PLAS, K=2, q_hi=(1,), quanta=(1, None), beta=(3, 1), max_batch=1))
    e.table.ensure(1, 0)
    e.table.svc[1] = 10
    e.register(0, [(1, 1, 0, 0, 0)])
    assert e.calls[1].q == 1
    e.table.ensure(2, 0)
    e.register(0, [(2, 2, 0, 0, 0)])
    promoted_at = None
    for t in range(100):
        e.demote_and_promote()
        if e.calls[1].q == 0 and promoted_at is None:
            promoted_at = t
        e.schedule(t)
    # W/T >= 3 with T = 10 needs W = 30 waiting steps
    assert promoted_at == 30
