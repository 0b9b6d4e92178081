"""Pins of the oracle's exact Eq. 2 ATLAS mode (reading R31).

Eq. 2: p(c_j) = 0 for a root, else max over the parents c_k of p(c_k) + t_k.  The
scalar ATLAS of Alg. 1 (l.4, l.11) instead hands every new call the program's longest observed
critical path.  Pins: a hand-worked fork (tests/golden/eq2_fork.json), a brute-force longest
path over every root-to-parent path of random DAGs (the definition Eq. 2 recurses on, P:L239
"the longest chain of accumulated service time leading to c_j"), and the two reductions the
SPEC lists (S:L286 chains; S:L635(c) joins whose parents hold the longest observed path)."""
import json
import os

import pytest

from autx_workload import dag_trace, random_tiny, mcts_mapreduce
from oracle.autellix import Config, simulate, Engine, ATLAS, ATLAS_EQ2

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "eq2_fork.json")


def test_eq2_fork_golden():
    g = json.load(open(GOLDEN))
    tr = dag_trace("eq2_fork", [g["trace"]], [0])
    c = g["config"]
    for pol, key in ((ATLAS_EQ2, "inh_eq2"), (ATLAS, "inh_atlas")):
        cfg = Config(policy=pol, K=c["K"], quanta=tuple(c["quanta"]), max_batch=c["max_batch"],
                     beta=tuple(c["beta"]))
        _, m = simulate(tr, cfg)
        got = {str(int(cid) & 0xFFFF): v for cid, v in m["inh"].items()}
        assert got == g[key], pol


def longest_path_priority(tr, c):
    """Brute force: enumerate every path root -> ... -> parent of c through the parent lists and
    take the largest sum of execution times (a call executes exactly its decode length)."""
    best = 0
    stack = [(int(k), int(tr.decode[k])) for k in tr.parents(c)]
    while stack:
        k, acc = stack.pop()
        best = max(best, acc)
        for j in tr.parents(k):
            stack.append((int(j), acc + int(tr.decode[j])))
    return best


@pytest.mark.parametrize("seed", range(60))
def test_eq2_is_longest_path(seed):
    tr = random_tiny(seed, max_programs=3, max_calls=6, max_decode=5, max_delay=3)
    bs = 1 + seed % 3
    cfg = Config(policy=ATLAS_EQ2, K=3, q_hi=(2, 5), quanta=(1, 2, None), max_batch=bs,
                 beta=[(1, 0), (2, 1)][seed % 2])
    _, m = simulate(tr, cfg)
    for c in range(tr.n_calls):
        assert m["inh"][int(tr.call_id[c])] == longest_path_priority(tr, c), (seed, c)


def logs(tr, cfg):
    log, m = simulate(tr, cfg)
    return [(r["t"], r["batch"], r["admit"], r["preempt"]) for r in log], m["inh"]


@pytest.mark.parametrize("seed", range(40))
def test_eq2_equals_scalar_on_chains(seed):
    """on chains the single-parent max is the scalar (both equal PLAS)."""
    tr = random_tiny(seed, dag=False, max_calls=5)
    base = dict(K=3, q_hi=(2, 5), quanta=(1, 2, None), max_batch=1 + seed % 2, beta=(2, 1))
    assert logs(tr, Config(policy=ATLAS_EQ2, **base)) == logs(tr, Config(policy=ATLAS, **base))


@pytest.mark.parametrize("seed", range(3))
def test_eq2_equals_scalar_on_map_reduce(seed):
    """S:L635(c): every reduce joins all of its program's maps, so its parents hold the longest
    observed path and Eq. 2 gives the scalar; maps are roots (0 in both)."""
    tr = mcts_mapreduce(n_programs=6, seed=100 + seed, frac_mcts=0.0)
    base = dict(K=8, q_hi=tuple(2 * 4 ** i for i in range(7)), quanta=(2, 6, 24, 96, 384, 1536, 6144, None),
                max_batch=64, beta=(2, 1))
    assert logs(tr, Config(policy=ATLAS_EQ2, **base)) == logs(tr, Config(policy=ATLAS, **base))


def test_eq2_differs_on_mcts():
    """MCTS evaluates depend on one expand each: Eq. 2 gives them their own thread's path while
    the scalar gives the program's longest, so once a batch limit staggers the threads (a
    shorter thread finishing after a longer one) inherited priorities differ, never upwards
    (p_eq2 <= p_scalar by induction over the DAG)."""
    tr = mcts_mapreduce(n_programs=4, seed=7, frac_mcts=1.0)
    base = dict(K=1, quanta=(None,), max_batch=4)
    _, a = logs(tr, Config(policy=ATLAS_EQ2, **base))
    _, b = logs(tr, Config(policy=ATLAS, **base))
    assert all(a[k] <= b[k] for k in a) and any(a[k] < b[k] for k in a)


def test_eq2_parent_must_be_completed():
    eng = Engine(Config(policy=ATLAS_EQ2, K=1, quanta=(None,), max_batch=2))
    eng.register(0, [(1, 0, 0, 0, 4)], {1: []})
    with pytest.raises(KeyError):
        eng.register(1, [(2, 0, 1, 0, 4)], {2: [1]})  # parent 1 is still active
