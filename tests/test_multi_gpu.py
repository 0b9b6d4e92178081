"""Multi-engine CUDA path against the oracle's lockstep multi-engine simulation:
per-engine decision logs and Alg. 2 routing decisions must be identical.  Two engines share one
B200 with their records exchanged over gloo (autx_route_pack / autx_route_apply); the one-call
collective autx_route (ncclAllGather on the library's communicator) runs as one engine on one
GPU, and as two engines when two GPUs exist."""
import pytest

from multi_harness import run_world, oracle_multi

pytestmark = pytest.mark.gpu

CFGS = [
    dict(policy="plas", K=2, q_hi=(1,), quanta=(1, None), max_batch=2, block_tokens=4, token_threshold=8),
    dict(policy="atlas", K=3, q_hi=(2, 5), quanta=(1, 2, None), beta=(2, 1), max_batch=3,
         block_tokens=4, token_threshold=10),
    dict(policy="atlas", K=8, q_hi=(2, 8, 32, 128, 512, 2048, 8192), quanta=(2, 6, 24, 96, 384, 1536, 6144, None),
         beta=(2, 1), max_batch=16, kv_budget=3000, token_threshold=2048),
]


@pytest.mark.parametrize("trace,seed,ci", [("tiny", 1, 0), ("tiny", 2, 1), ("tiny", 9, 1),
                                           ("chatbot", 0, 2), ("mcts", 0, 2)])
def test_two_engines_match_oracle(tmp_path, trace, seed, ci):
    res = run_world(tmp_path, True, trace, seed, CFGS[ci])
    want, routes = oracle_multi(trace, seed, CFGS[ci])
    for r in range(2):
        assert res[r]["log"] == want[r], f"engine {r}"
        assert [x for x in res[r]["routes"] if x[1]] == [x for x in routes if x[1]]


def test_two_engines_golden_route(tmp_path):
    """Two CUDA engines on the hand-derived trace (tests/golden/route_2engine.json): Alg. 2
    routes (load after completions, first-long-call pin) and decisions equal the golden."""
    from multi_harness import golden_route
    cfg, routes, logs = golden_route()
    res = run_world(tmp_path, True, "golden_route", 0, cfg)
    for r in range(2):
        assert res[r]["log"] == logs[r], f"engine {r}"
        assert [x for x in res[r]["routes"] if x[1]] == routes


@pytest.mark.parametrize("router", ["least_used", "round_robin"])
@pytest.mark.parametrize("trace,seed,ci", [("tiny", 2, 1), ("chatbot", 0, 2)])
def test_two_engines_comparator_routers(tmp_path, router, trace, seed, ci):
    """The §6.4 comparators in k_route: routes and decisions equal the oracle's
    simulate_multi(router=...)."""
    res = run_world(tmp_path, True, trace, seed, CFGS[ci], router=router)
    want, routes = oracle_multi(trace, seed, CFGS[ci], router=router)
    for r in range(2):
        assert res[r]["log"] == want[r], f"engine {r}"
        assert [x for x in res[r]["routes"] if x[1]] == [x for x in routes if x[1]]


@pytest.mark.parametrize("trace,seed,ci", [("tiny", 2, 1), ("mcts", 0, 2)])
def test_route_collective_single_engine(tmp_path, trace, seed, ci):
    """autx_route with a one-rank NCCL communicator: header kernel, ncclAllGather, k_route; the
    decisions and (trivial) routes equal simulate_multi with G = 1."""
    res = run_world(tmp_path, "nccl", trace, seed, CFGS[ci], world=1)
    want, routes = oracle_multi(trace, seed, CFGS[ci], world=1)
    assert res[0]["log"] == want[0]
    assert [x for x in res[0]["routes"] if x[1]] == [x for x in routes if x[1]]


@pytest.mark.parametrize("trace,seed,ci", [("tiny", 2, 1), ("chatbot", 0, 2), ("golden_route", 0, None)])
def test_two_engines_route_collective(tmp_path, trace, seed, ci):
    """Two engines on two GPUs through autx_route (NCCL all-gather over NVLink)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (NCCL refuses two ranks on one device)")
    if trace == "golden_route":
        from multi_harness import golden_route
        cfg, routes, logs = golden_route()
        res = run_world(tmp_path, "nccl", trace, 0, cfg)
        for r in range(2):
            assert res[r]["log"] == logs[r]
            assert [x for x in res[r]["routes"] if x[1]] == routes
        return
    res = run_world(tmp_path, "nccl", trace, seed, CFGS[ci])
    want, routes = oracle_multi(trace, seed, CFGS[ci])
    for r in range(2):
        assert res[r]["log"] == want[r], f"engine {r}"
        assert [x for x in res[r]["routes"] if x[1]] == [x for x in routes if x[1]]
