"""Multi-engine oracle pinned to a hand-derived two-engine trace (tests/golden/route_2engine.json):
the Alg. 2 routes and both engines' decisions.  The trace is built so that the
routing depends on the two points the other oracle tests leave open:
  * the load snapshot is taken AFTER the step's completions (reading R23): taken before them,
    d0 and a1 at t=1 go the other way round and D is pinned to the other engine;
  * the pin is set by the program's first long call and then holds for its later long calls
    even against the load (Alg. 2 l.5-10): d2 at t=6 goes to the busier pinned engine."""
import json
import os

from autx_workload import dag_trace
from oracle.autellix import Config, simulate_multi, route

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "route_2engine.json")


def golden_trace_and_config():
    g = json.load(open(GOLDEN))
    tr = dag_trace("route_2engine", [dict(decode=p["decode"], prefill=p["prefill"], delay=p["delay"],
                                          parents=p["parents"]) for p in g["programs"]], [0] * len(g["programs"]))
    c = g["config"]
    cfg = Config(policy=c["policy"], K=c["K"], q_hi=tuple(c["q_hi"]), quanta=tuple(c["quanta"]),
                 beta=tuple(c["beta"]), max_batch=c["max_batch"], token_threshold=c["token_threshold"])
    return g, tr, cfg


def test_two_engine_golden_routes_and_batches():
    g, tr, cfg = golden_trace_and_config()
    logs, routes = simulate_multi(tr, cfg, 2)
    assert [[t, list(c), list(d)] for t, c, d in routes if c] == g["routes"]
    for e in range(2):
        got = [[r["t"], r["batch"], r["admit"], r["preempt"]] for r in logs[e] if r["batch"] or r["preempt"]]
        assert got == g["batches"][e], f"engine {e}"


def test_golden_discriminates_the_snapshot_point_and_the_pin():
    """The golden's t=1 and t=6 routings, recomputed from the loads the derivation states:
    after the completions ([1,1]) vs before them ([2,1]); pinned vs least-loaded for d2."""
    pins = {}
    assert route([(0, 0, 3000), (65537, 1, 201)], [1, 1], pins) == [0, 1] and pins == {0: 0}
    pins_before = {}
    assert route([(0, 0, 3000), (65537, 1, 201)], [2, 1], pins_before) == [1, 0] and pins_before == {0: 1}
    assert route([(1, 0, 3011), (2, 0, 3011), (262144, 4, 100)], [0, 0], {0: 0}) == [0, 0, 1]
    assert route([(2, 0, 3011)], [1, 0], {}) == [1]  # unpinned, d2 would take the lighter engine
