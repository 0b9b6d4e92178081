"""N > 1 host-side path on CPU: world_size-2 gloo run of the multi-engine lockstep driver
(record all-gather, replicated arrivals, Alg. 2 routing, global readiness) with an
oracle-backed stand-in scheduler, against the oracle's own lockstep simulation."""
import pytest

from multi_harness import run_world, oracle_multi

CFGS = [
    dict(policy="plas", K=2, q_hi=(1,), quanta=(1, None), max_batch=2, block_tokens=4, token_threshold=8),
    dict(policy="atlas", K=3, q_hi=(2, 5), quanta=(1, 2, None), beta=(2, 1), max_batch=3,
         block_tokens=4, token_threshold=10),
]


@pytest.mark.parametrize("seed,ci", [(1, 0), (2, 1), (5, 1)])
def test_gloo_world2_matches_oracle_lockstep(tmp_path, seed, ci):
    res = run_world(tmp_path, False, "tiny", seed, CFGS[ci])
    want, routes = oracle_multi("tiny", seed, CFGS[ci])
    for r in range(2):
        assert res[r]["log"] == want[r]
        got_routes = [x for x in res[r]["routes"] if x[1]]
        assert got_routes == [x for x in routes if x[1]]


def test_gloo_world2_golden_route(tmp_path):
    """The hand-derived two-engine trace (tests/golden/route_2engine.json) through the driver's
    host protocol: routes and per-engine decisions equal the golden, not only the oracle."""
    from multi_harness import golden_route
    cfg, routes, logs = golden_route()
    res = run_world(tmp_path, False, "golden_route", 0, cfg)
    for r in range(2):
        assert res[r]["log"] == logs[r]
        assert [x for x in res[r]["routes"] if x[1]] == routes


@pytest.mark.parametrize("router", ["least_used", "round_robin"])
def test_gloo_world2_comparator_routers(tmp_path, router):
    res = run_world(tmp_path, False, "tiny", 2, CFGS[1], router=router)
    want, routes = oracle_multi("tiny", 2, CFGS[1], router=router)
    for r in range(2):
        assert res[r]["log"] == want[r]
        assert [x for x in res[r]["routes"] if x[1]] == [x for x in routes if x[1]]
