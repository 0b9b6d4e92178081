"""Oracle pins: SPEC.md worked examples for each operation (values the spec states,
each [PAPER]/[TRIVIAL]/[DERIVED] example re-derived by hand here)."""
import pytest

from oracle.autellix import (Engine, Config, ProgramTable, route, PLAS, ATLAS, MLFQ, FCFS,
                             ceil_div)


def eng(**kw):
    base = dict(policy=PLAS, K=3, q_hi=(2, 8), quanta=(2, 6, None), max_batch=2)
    base.update(kw)
    return Engine(Config(**base))


def test_placement_spec_examples():
    """bounds {[0,2),[2,8),[8,inf)}: priority 0 -> Q1, 5 -> Q2."""
    e = eng()
    assert e.place(0) == 0
    assert e.place(5) == 1
    assert e.place(1) == 0 and e.place(2) == 1 and e.place(7) == 1 and e.place(8) == 2  # half-open
    assert e.place(10 ** 9) == 2
    assert eng(policy=MLFQ).place(100) == 0 and eng(policy=FCFS).place(100) == 0


def test_plas_table_spec_examples():
    """first call 0; A after 4 steps -> 4; {3,3} -> 6; 4+3 -> 7."""
    t = ProgramTable()
    t.ensure(1, 0)
    assert t.svc[1] == 0
    t.apply_completion(PLAS, 1, 4, 0, 0, 4)
    assert t.svc[1] == 4
    t.apply_completion(PLAS, 1, 3, 4, 0, 7)
    assert t.svc[1] == 7
    t.ensure(2, 0)
    t.apply_completion(PLAS, 2, 3, 0, 0, 3)
    t.apply_completion(PLAS, 2, 3, 0, 0, 6)
    assert t.svc[2] == 6


def test_atlas_table_spec_examples():
    """S:L291 fork: root 3 -> {5, 2} gives scalar 8, not 10.  S:L299-300: scalar 8 +
    completion (inh 3, exec 2) stays 8; (inh 8, exec 4) -> 12."""
    t = ProgramTable()
    t.ensure(1, 0)
    t.apply_completion(ATLAS, 1, 3, 0, 0, 3)          # root
    t.apply_completion(ATLAS, 1, 5, 3, 0, 8)          # child inherits 3
    t.apply_completion(ATLAS, 1, 2, 3, 0, 8)
    assert t.svc[1] == 8
    t.apply_completion(ATLAS, 1, 2, 3, 0, 9)
    assert t.svc[1] == 8
    t.apply_completion(ATLAS, 1, 4, 8, 0, 13)
    assert t.svc[1] == 12


def _one_call_engine(policy=PLAS, beta=(1, 0), **kw):
    e = eng(policy=policy, beta=beta, **kw)
    e.register(0, [(10, 1, 0, 0, 0)])
    return e, e.calls[10]


def test_demotion_spec_examples():
    """quantum 2 and ran 2 -> demoted one level; queue K exhausting its quantum
    stays in K with a refreshed quantum; quantum 4, ran 3 -> not demoted."""
    e, c = _one_call_engine(K=3, q_hi=(2, 8), quanta=(2, 4, 3))
    for t in range(2):
        e.demote_and_promote()
        e.schedule(t)
    assert c.quanta == 0
    e.demote_and_promote()
    assert c.q == 1 and c.quanta == 4
    for t in range(3):
        e.schedule(t)
    e.demote_and_promote()
    assert c.q == 1 and c.quanta == 1          # ran 3 of 4: not demoted
    e.schedule(9)
    e.demote_and_promote()
    assert c.q == 2 and c.quanta == 3
    for t in range(3):
        e.schedule(t)
    e.demote_and_promote()
    assert c.q == 2 and c.quanta == 3          # clamped at K, quantum refreshed


def test_anti_starvation_spec_examples():
    """p.wait=9, c.wait=1, p.service=4, c.model_time=1, beta=2 -> 10/5 = 2 >= 2 ->
    promoted with c.wait and c.model_time reset.  S:L331: 0/0 -> none.  S:L329: beta=inf
    -> none."""
    e, c = _one_call_engine(beta=(2, 1))
    e.table.pwait[1] = 9
    e.table.svc[1] = 4
    c.q, c.quanta, c.wait, c.mtime = 2, None, 1, 1
    e.demote_and_promote()
    assert (c.q, c.quanta, c.wait, c.mtime) == (0, 2, 0, 0)
    # just below the threshold: 9/5 < 2 -> stays
    e2, c2 = _one_call_engine(beta=(2, 1))
    e2.table.pwait[1] = 8
    e2.table.svc[1] = 4
    c2.q, c2.quanta, c2.wait, c2.mtime = 2, None, 1, 1
    e2.demote_and_promote()
    assert c2.q == 2 and c2.wait == 1
    # 0/0 never promotes
    e3, c3 = _one_call_engine(beta=(2, 1))
    c3.q = 1
    e3.demote_and_promote()
    assert c3.q == 1
    # beta = infinity never promotes
    e4, c4 = _one_call_engine(beta=(1, 0))
    e4.table.pwait[1] = 10 ** 6
    c4.q = 2
    e4.demote_and_promote()
    assert c4.q == 2
    # W>0, T=0 -> ratio infinite -> promotes for any finite beta
    e5, c5 = _one_call_engine(beta=(1000, 1))
    c5.q, c5.wait = 2, 1
    e5.demote_and_promote()
    assert c5.q == 0


def test_form_batch_spec_examples():
    """BS=2, Q1={C1,D1}, Q2={A2,B2} -> {C1,D1}; empty -> empty;
    BS=2, Q1={X}, Q2={Y,Z} -> {X,Y}."""
    e = eng(K=2, q_hi=(1,), quanta=(1, None))
    assert e.schedule(0)["batch"] == []
    e.table.ensure(1, 0); e.table.svc[1] = 4
    e.table.ensure(2, 0); e.table.svc[2] = 4
    e.register(0, [(100, 1, 0, 0, 0), (200, 2, 0, 0, 0), (300, 3, 0, 0, 0), (400, 4, 0, 0, 0)])
    assert e.schedule(0)["batch"] == [300, 400]
    e = eng(K=2, q_hi=(1,), quanta=(1, None))
    e.table.ensure(2, 0); e.table.svc[2] = 5
    e.table.ensure(3, 0); e.table.svc[3] = 5
    e.register(0, [(1, 1, 0, 0, 0), (2, 2, 0, 0, 0), (3, 3, 0, 0, 0)])
    assert e.schedule(0)["batch"] == [1, 2]


def test_kv_cutoff_stops_at_first_misfit():
    """Alg. 1 l.36-37 `break`: a smaller later call is NOT backfilled (reading R13)."""
    e = eng(K=1, q_hi=(), quanta=(None,), max_batch=3, kv_budget=4, block_tokens=4,
            block_bytes=1000)
    # kvb = ceil((tok + exec + 1)/4): tok 7 -> 2, tok 11 -> 3, tok 0 -> 1
    e.register(0, [(1, 1, 0, 0, 7), (2, 2, 0, 0, 11), (3, 3, 0, 0, 0)])
    r = e.schedule(0)
    # call 2 misfits (2+3 > 4); call 3 would fit (2+1 <= 4) but is not backfilled
    assert r["batch"] == [1] and r["kv_blocks"] == 2
    e.complete(1, [1])
    r = e.schedule(1)
    assert r["batch"] == [2, 3] and r["kv_blocks"] == 4 and r["admit"] == [2, 3]
    assert r["preempt"] == [] and r["swap_in"] == 0  # fresh calls: allocation, not swap-in
    # KV grows as the call decodes: call 3 now needs ceil((0+1+1)/4) = 1, call 2 ceil(13/4)=4
    r = e.schedule(2)
    assert r["batch"] == [2] and r["preempt"] == [3] and r["swap_out"] == 1 * 1000


def test_preempt_swap_bytes_closed_form():
    """A call preempted after one step holds ceil((input+1)/bt) blocks; swapping it
    back in moves the same bytes (reading R14/R15)."""
    e = Engine(Config(policy=PLAS, K=2, q_hi=(1,), quanta=(1, None), max_batch=1,
                      block_tokens=16, block_bytes=2 << 20))
    e.register(0, [(1, 1, 0, 0, 20)])
    r0 = e.schedule(0)
    assert r0["batch"] == [1]
    e.register(1, [(2, 2, 1, 1, 5)])
    e.demote_and_promote()            # call 1 exhausted its quantum -> Q2
    r1 = e.schedule(1)
    assert r1["batch"] == [2] and r1["preempt"] == [1]
    assert r1["swap_out"] == ceil_div(20 + 1, 16) * (2 << 20)
    e.complete(2, [2])
    e.demote_and_promote()
    r2 = e.schedule(2)
    assert r2["batch"] == [1] and r2["admit"] == [1]
    assert r2["swap_in"] == r1["swap_out"]


def test_routing_spec_examples():
    """1 engine -> 0; long call of a program pinned to engine 2 -> 2
    regardless of load; short call with loads {5,2,7} -> 1.  Ties -> lowest id."""
    assert route([(1, 1, 100)], [3], {}) == [0]
    assert route([(1, 7, 3000)], [0, 0, 99, 0], {7: 2}) == [2]
    assert route([(1, 7, 100)], [5, 2, 7], {}) == [1]
    assert route([(1, 7, 100)], [4, 4, 4], {}) == [0]
    # first long call pins (Alg. 2 l.10); later long calls follow the pin; loads increment
    pins, loads = {}, [1, 0]
    assert route([(1, 9, 5000), (2, 9, 100), (3, 9, 5000)], loads, pins) == [1, 0, 1]
    assert pins == {9: 1} and loads == [2, 2]
    # threshold is inclusive: LEN <= 2048 is short (Alg. 2 l.2, reading R21)
    pins = {}
    route([(1, 5, 2048)], [0, 0], pins)
    assert pins == {}
    with pytest.raises(ValueError):
        route([(1, 1, 1)], [], {})
