"""GPU parity for multi-step scheduling with over-provisioning (SURVEY §8(f) item 1, P:L292,
reading R32): the CUDA path (window steps: k_window + finalize; scheduling points: the full
chain with a BS + X resident set; demotion deferred through QF_DEM) against the oracle, list for
list (batch, standby, admit, preempt) with the swap and KV ledgers, including the KV block
allocator with a byte-pattern round trip of every swapped block."""
import json
import os

import pytest

from autx_workload import random_tiny, chatbot, react
from autx_workload.gen import dag_trace
from oracle.autellix import Config, simulate, spec_ladder_config, FCFS, MLFQ, PLAS, ATLAS, CapacityError

pytestmark = pytest.mark.gpu

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "multistep.json")))


def make_sched(cfg, **kw):
    from paper_2502_13965_b200 import Scheduler
    args = dict(policy=cfg.policy, K=cfg.K, q_hi=cfg.q_hi, quanta=cfg.quanta, beta=cfg.beta,
                max_batch=cfg.max_batch, kv_budget=cfg.kv_budget, block_tokens=cfg.block_tokens,
                max_calls=kw.pop("max_calls", 1 << 14), max_programs=kw.pop("max_programs", 1 << 12),
                token_threshold=cfg.token_threshold, sched_every=cfg.sched_every,
                overprovision=cfg.overprovision)
    args.update(kw)
    return Scheduler(**args)


def rec_tuple(r, sw_out, sw_in, kvb):
    return (r["t"], r["batch"], r.get("standby", []), r["admit"], r["preempt"], r[sw_out], r[sw_in], r[kvb])


def oracle_records(tr, cfg):
    cfg.block_bytes = 1
    log, _ = simulate(tr, cfg, check_formulations=False)
    return [rec_tuple(r, "swap_out", "swap_in", "kv_blocks") for r in log if r["batch"] or r["preempt"]]


def gpu_records(tr, cfg, **kw):
    from paper_2502_13965_b200 import TraceDriver
    s = make_sched(cfg, **kw)
    log = TraceDriver(tr, s).run()
    s.close()
    return [rec_tuple(r, "swap_out_blocks", "swap_in_blocks", "kv_blocks") for r in log if r["batch"] or r["preempt"]]


def assert_same(got, want):
    assert len(got) == len(want), f"{len(got)} vs {len(want)} steps"
    for g, w in zip(got, want):
        assert g == w, f"step {w[0]}: gpu {g} != oracle {w}"


@pytest.mark.parametrize("case", G["cases"], ids=[c["name"] for c in G["cases"]])
def test_golden_multistep(case):
    progs = [dict(decode=p["decode"], parents=[[]] * len(p["decode"])) for p in case["programs"]]
    tr = dag_trace(case["name"], progs, [p["arrival"] for p in case["programs"]])
    c = dict(case["config"])
    c["q_hi"], c["quanta"] = tuple(c["q_hi"]), tuple(c["quanta"])
    got = gpu_records(tr, Config(**c).check())
    prog = lambda cids: [int(x) >> 16 for x in cids]
    got = [dict(t=g[0], batch=prog(g[1]), standby=prog(g[2]), admit=prog(g[3]), preempt=prog(g[4])) for g in got]
    assert got == case["steps"]


LADDERS = [dict(K=1, q_hi=(), quanta=(None,)), dict(K=2, q_hi=(1,), quanta=(1, None)),
           dict(K=3, q_hi=(2, 5), quanta=(1, 2, None)), dict(K=4, q_hi=(1, 3, 6), quanta=(2, 1, 3, 2))]
NX = [(2, 1), (3, 2), (2, 0), (4, 1), (1, 2), (3, 0)]


def tiny_cfg(i, policy):
    N, X = NX[i % len(NX)]
    return Config(policy=policy, max_batch=1 + i % 3, kv_budget=(None, 8, 12)[(i // 3) % 3],
                  beta=((1, 0), (2, 1), (1, 2), (5, 3))[(i // 9) % 4], block_tokens=4,
                  sched_every=N, overprovision=X, **LADDERS[i % 4])


@pytest.mark.parametrize("seed", range(150))
def test_random_tiny_multistep(seed):
    tr = random_tiny(seed)
    for p, policy in enumerate((FCFS, MLFQ, PLAS, ATLAS)):
        cfg = tiny_cfg(seed * 4 + p, policy)
        try:
            want = oracle_records(tr, cfg)
        except CapacityError:
            from paper_2502_13965_b200 import AutxError
            with pytest.raises(AutxError) as e:
                gpu_records(tr, tiny_cfg(seed * 4 + p, policy))
            assert e.value.code == 4
            continue
        except ValueError:
            continue
        assert_same(gpu_records(tr, tiny_cfg(seed * 4 + p, policy)), want)


@pytest.mark.parametrize("N,X", [(4, 8), (2, 0), (1, 8)])
def test_chatbot_slice_multistep(N, X):
    cfg = lambda: Config(**{**spec_ladder_config(PLAS, max_batch=32, kv_budget=2400).__dict__,
                            "sched_every": N, "overprovision": X})
    tr = chatbot(300)
    assert_same(gpu_records(tr, cfg()), oracle_records(tr, cfg()))


@pytest.mark.parametrize("N,X", [(4, 16), (8, 16)])
def test_react_slice_multistep_with_kv_allocator(N, X):
    """ReAct-shaped programs with the KV block allocator: lists and ledgers equal the oracle's,
    and the multi-step schedule swaps fewer blocks than the every-step one."""
    def cfg(n, x):
        return Config(**{**spec_ladder_config(PLAS, max_batch=64, kv_budget=4000).__dict__,
                         "sched_every": n, "overprovision": x})
    tr = react(400)
    want = oracle_records(tr, cfg(N, X))
    got = gpu_records(tr, cfg(N, X), n_gpu_blocks=4000, max_blocks_per_call=4096, host_pages=1 << 16)
    assert_same(got, want)
    plain = oracle_records(tr, cfg(1, 0))
    assert sum(g[5] + g[6] for g in got) < sum(w[5] + w[6] for w in plain)


def test_kv_round_trip_bytes_multistep():
    """Standby calls keep their blocks, window-step evictions and scheduling-point preemptions
    swap out only calls with KV content: after every step each batch call's blocks hold exactly
    the bytes written when it ran before (SM-driven swap)."""
    import torch
    from paper_2502_13965_b200 import TraceDriver
    tr = chatbot(120)
    L, chunk, P = 2, 1024, 2400
    mk = lambda: Config(**{**spec_ladder_config(PLAS, max_batch=16, kv_budget=P).__dict__,
                           "sched_every": 3, "overprovision": 4})
    want = oracle_records(tr, mk())
    s = make_sched(mk(), n_gpu_blocks=P, max_blocks_per_call=4096, host_pages=1 << 14)
    kpools = [torch.zeros(P, chunk // 4, dtype=torch.int32, device="cuda") for _ in range(L)]
    vpools = [torch.zeros(P, chunk // 4, dtype=torch.int32, device="cuda") for _ in range(L)]
    host = torch.zeros((1 << 14) * L * 2 * chunk // 4, dtype=torch.int32).pin_memory()
    d = TraceDriver(tr, s)
    written, got = {}, []

    def pat(cid, j, l, kv):
        return (cid * 1000003 + j * 101 + l * 7 + kv) & 0x7FFFFFFF

    while not d.finished():
        if len(d.pending) == 0 and s.num_active() == 0 and d.t not in d.ready:
            d.t = min(d.ready)
        rec = d.step()
        st = s.kv_swap([p.data_ptr() for p in kpools], [p.data_ptr() for p in vpools], chunk,
                       host.data_ptr(), host.numel() * 4, 0)
        assert st.bytes_d2h == rec["swap_out_blocks"] * L * 2 * chunk
        assert st.bytes_h2d == rec["swap_in_blocks"] * L * 2 * chunk
        offs, blks = s.block_table_host()
        for i, cid in enumerate(rec["batch"]):
            mine = blks[offs[i]:offs[i + 1]]
            w = written.get(cid, 0)
            assert len(mine) >= w
            for l in range(L):
                for kv, pools in ((0, kpools), (1, vpools)):
                    if w:
                        idx = torch.tensor([int(b) for b in mine[:w]], device="cuda", dtype=torch.long)
                        exp = torch.tensor([pat(cid, j, l, kv) for j in range(w)], device="cuda", dtype=torch.int32)
                        assert bool((pools[l][idx] == exp[:, None]).all()), f"KV corrupted at t={rec['t']}"
                    if len(mine) > w:
                        idx = torch.tensor([int(b) for b in mine[w:]], device="cuda", dtype=torch.long)
                        val = torch.tensor([pat(cid, j, l, kv) for j in range(w, len(mine))], device="cuda",
                                           dtype=torch.int32)
                        pools[l][idx] = val[:, None].expand(-1, chunk // 4)
            written[cid] = len(mine)
        got.append(rec_tuple(rec, "swap_out_blocks", "swap_in_blocks", "kv_blocks"))
    got = [g for g in got if g[1] or g[4]]
    assert_same(got, want)
    s.close()


@pytest.mark.parametrize("kv", [None, 3000])
def test_multistep_exact_eq2(kv):
    """Exact Eq. 2 inheritance (R31) under multi-step scheduling: DAG arrivals registered in window
    steps inherit from parents completed mid-window."""
    from autx_workload import mcts_mapreduce
    from oracle.autellix import ATLAS_EQ2
    cfg = lambda: Config(**{**spec_ladder_config(ATLAS_EQ2, max_batch=16, kv_budget=kv).__dict__,
                            "sched_every": 3, "overprovision": 4})
    tr = mcts_mapreduce(12)
    extra = dict(n_gpu_blocks=kv, max_blocks_per_call=4096, host_pages=1 << 14) if kv else {}
    assert_same(gpu_records(tr, cfg(), **extra), oracle_records(tr, cfg()))


@pytest.mark.parametrize("N,X", [(3, 4), (1, 4)])
def test_multistep_with_compaction(N, X):
    """The resident list (batch + standby) survives device compaction (k_remap_prev)."""
    cfg = lambda: Config(**{**spec_ladder_config(PLAS, max_batch=16, kv_budget=2400).__dict__,
                            "sched_every": N, "overprovision": X})
    tr = chatbot(200)
    assert_same(gpu_records(tr, cfg(), max_calls=400, n_gpu_blocks=2400, max_blocks_per_call=4096,
                            host_pages=1 << 14), oracle_records(tr, cfg()))


def test_config_errors():
    from paper_2502_13965_b200 import AutxError
    base = spec_ladder_config(PLAS, max_batch=16)
    with pytest.raises(AutxError):
        make_sched(Config(**{**base.__dict__, "sched_every": 2}), order_mode=1)
    with pytest.raises(AutxError):
        make_sched(Config(**{**base.__dict__, "overprovision": 2040}))
