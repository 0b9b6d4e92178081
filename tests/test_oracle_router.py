"""Router locality economics: the §6.4 comparators and the
program-prefix cache model behind Alg. 2's short/long split (§4.3; reading R34), pinned
to hand examples, and the directional Fig. 14 result."""
from autx_workload import dag_trace, chatbot
from oracle.autellix import (Config, PLAS, PrefixCache, route, route_least_used, route_round_robin,
                             simulate_multi, spec_ladder_config)


def test_round_robin_is_cyclic_across_steps():
    st = {"next": 0}
    assert route_round_robin([1, 2, 3, 4, 5], 3, st) == [0, 1, 2, 0, 1]
    assert route_round_robin([6], 3, st) == [2] and st["next"] == 0


def test_least_used_ignores_length_and_pins():
    loads = [3, 1, 1]
    assert route_least_used([(1, 7, 5000), (2, 7, 5000), (3, 7, 100)], loads) == [1, 2, 1]
    assert loads == [3, 3, 2]
    # Alg. 2 on the same calls with program 7 pinned to engine 0 keeps the long calls there
    assert route([(1, 7, 5000), (2, 7, 5000), (3, 7, 100)], [3, 1, 1], {7: 0}) == [0, 0, 1]


def test_prefix_cache_by_hand():
    """Chain a (prompt 100, decodes 10) -> b (prompt 20, 5) -> c (prompt 30): inputs 100, 130,
    165.  On one engine b reuses a's 110 tokens and c reuses b's 135: prefill 100 + 20 + 30;
    b on another engine recomputes all 130."""
    same = PrefixCache(2)
    assert same.admit(0, 9, 100, 100) == 0
    same.done(0, 9, 100, 10)
    assert same.admit(0, 9, 130, 20) == 110
    same.done(0, 9, 130, 5)
    assert same.admit(0, 9, 165, 30) == 135
    assert same.prefill == 150
    other = PrefixCache(2)
    other.admit(0, 9, 100, 100)
    other.done(0, 9, 100, 10)
    assert other.admit(1, 9, 130, 20) == 0 and other.prefill == 230


def test_locality_routing_saves_prefill_directional():
    """S:L639 / Fig. 14: four engines, ShareGPT-shaped chains whose contexts outgrow the 2048-token
    threshold: Alg. 2 recomputes strictly fewer prompt tokens and reuses a strictly larger share of
    the long calls' context than Round Robin and Least Used on the same trace."""
    tr = chatbot(240, seed=7, rate=0.5)
    cfg = spec_ladder_config(PLAS, max_batch=16)
    res = {}
    for router in ("locality", "least_used", "round_robin"):
        cache = PrefixCache(4)
        simulate_multi(tr, cfg, 4, router=router, cache=cache)
        long = [(i, r) for i, r in cache.hits if i > cfg.token_threshold]
        res[router] = (cache.prefill, sum(r for _, r in long) / sum(i for i, _ in long))
    assert res["locality"][0] < min(res["least_used"][0], res["round_robin"][0])
    assert res["locality"][1] > max(res["least_used"][1], res["round_robin"][1])
