"""Oracle pins: the paper's Fig. 2 worked example and its brute-force bound."""
import json
import os
from functools import lru_cache

import pytest

from autx_workload import fig2
from oracle.autellix import (FCFS, MLFQ, PLAS, ATLAS, fig2_config, simulate, gantt_strings,
                             Config)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig2.json")))
NAMES = "ABCD"


def run(policy):
    tr = fig2()
    log, m = simulate(tr, fig2_config(policy))
    g = gantt_strings(tr, m["gantt"])
    return tr, log, m, {NAMES[p]: s for p, s in g.items()}


@pytest.mark.parametrize("policy", [FCFS, MLFQ, PLAS, ATLAS])
def test_fig2_total_wait_matches_paper(policy):
    _, _, m, _ = run(policy)
    assert m["total_wait"] == GOLD["total_wait"][policy]


@pytest.mark.parametrize("policy", [FCFS, MLFQ, PLAS])
def test_fig2_gantt(policy):
    _, _, _, g = run(policy)
    assert g == GOLD["gantt"][policy]


@pytest.mark.parametrize("policy", [FCFS, MLFQ, PLAS])
def test_fig2_per_call_waits(policy):
    """Per-call waiting derived from the Gantt: steps active but not running."""
    _, _, _, g = run(policy)
    dec = GOLD["trace"]
    waits = {}
    for prog, s in g.items():
        # a call is active from the end of its predecessor (or t=0) until it finishes
        start = 0
        for k, d in enumerate(dec[prog]):
            ch = str(k + 1)
            last = s.rindex(ch)
            w = (last + 1 - start) - d
            if w:
                waits[f"{prog}{k+1}"] = w
            start = last + 1
    assert waits == GOLD["per_call_wait"][policy]


def test_fig2_prose_constraints():
    """Text pins: FCFS delays C and D until t=3,4; MLFQ preempts A and B's long
    calls and runs A/B's later calls over t=6-12, delaying D; PLAS
    prioritises C and D over A and B's subsequent calls."""
    _, _, _, g = run(FCFS)
    assert g["C"].index("1") == 3 and g["D"].index("1") == 4
    _, _, _, g = run(MLFQ)
    # preemption of A1 and B1 after their first quantum
    assert g["A"][:2] == "1." and g["B"][:2] == "1."
    # D's single call is delayed until after A's and B's later calls at t=6-12
    assert g["D"].rindex("1") == 12
    later_ab = [t for t in range(6, 13) if (t < len(g["A"]) and g["A"][t] not in ".1")
                or (t < len(g["B"]) and g["B"][t] not in ".1")]
    assert len(later_ab) >= 6
    _, _, _, g = run(PLAS)
    # C's second call and D run before A's and B's second calls
    assert g["C"].index("2") < g["A"].index("2") and g["D"].rindex("1") < g["A"].index("2")


def fig2_bruteforce_opt():
    """Minimum total waiting over ALL preemptive schedules (chains, BS=2, no delays):
    exhaustive DP.  State = per program (call index, steps left in that call)."""
    dec = [tuple(v) for v in GOLD["trace"].values()]
    BS = GOLD["max_batch"]

    @lru_cache(maxsize=None)
    def best(state):
        active = [i for i, (k, _) in enumerate(state) if k < len(dec[i])]
        if not active:
            return 0
        from itertools import combinations
        res = None
        for chosen in combinations(active, min(BS, len(active))):
            nxt = list(state)
            for i in chosen:
                k, left = nxt[i]
                left -= 1
                nxt[i] = (k + 1, dec[i][k + 1] if k + 1 < len(dec[i]) else 0) if left == 0 else (k, left)
            cost = len(active) - len(chosen) + best(tuple(nxt))
            res = cost if res is None else min(res, cost)
        return res

    return best(tuple((0, d[0]) for d in dec))


def test_fig2_bruteforce_bound():
    opt = fig2_bruteforce_opt()
    assert opt == GOLD["brute_force_optimum"]
    assert opt <= GOLD["total_wait"]["plas"] <= GOLD["total_wait"]["fcfs"]


def test_fig2_chain_closed_form():
    """For chains with no interrupts, total waiting = sum over programs of
    (finish - arrival - total decode steps)."""
    for pol in (FCFS, MLFQ, PLAS):
        tr, _, m, _ = run(pol)
        dec = GOLD["trace"]
        cf = sum(m["finish"][p] - 0 - sum(dec[NAMES[p]]) for p in range(4))
        assert cf == m["total_wait"]


def test_fig2_spec_ladder_and_beta_sensitivity():
    """Derived regression values (independent prototype): the
    SPEC default ladder gives 11/11, and beta=2 moves MLFQ to 16 and PLAS to 14, while
    beta>=4 keeps 18/12."""
    tr = fig2()
    from oracle.autellix import spec_ladder_config
    for pol in (MLFQ, PLAS):
        cfg = spec_ladder_config(pol, max_batch=2, beta=(1, 0))
        assert simulate(tr, cfg)[1]["total_wait"] == 11
    for pol, want2 in ((MLFQ, 16), (PLAS, 14)):
        c = fig2_config(pol)
        c.beta = (2, 1)
        assert simulate(tr, c)[1]["total_wait"] == want2
        c.beta = (4, 1)
        assert simulate(tr, c)[1]["total_wait"] == GOLD["total_wait"][pol]


def test_atlas_dag_fixture():
    from autx_workload import atlas_dag_fixture
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "atlas_dag.json")))
    tr = atlas_dag_fixture()
    name = {int(c): f"P{int(c) >> 16}.{int(c) & 0xffff}" for c in tr.call_id}
    for pol in (PLAS, ATLAS):
        cfg = Config(policy=pol, K=3, q_hi=(2, 6), quanta=(2, 4, None), max_batch=2)
        log, m = simulate(tr, cfg)
        assert m["total_wait"] == gold["total_wait"][pol]
        if pol == ATLAS:
            got = [[name[c] for c in r["batch"]] for r in log if r["batch"]]
            assert got == gold["atlas_batches"]
