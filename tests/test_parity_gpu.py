"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, decision for decision
(batch, admit, preempt, swap blocks, KV blocks) and state for state, on seeded traces.
All comparisons are exact (integer method)."""
import numpy as np
import pytest

from autx_workload import fig2, random_tiny, atlas_dag_fixture, chatbot, react, mcts_mapreduce
from oracle.autellix import (Config, Engine, Workload, simulate, fig2_config, spec_ladder_config,
                             FCFS, MLFQ, PLAS, ATLAS, ATLAS_EQ2, CapacityError)

pytestmark = pytest.mark.gpu


def make_sched(cfg: Config, **kw):
    from paper_2502_13965_b200 import Scheduler
    args = dict(policy=cfg.policy, K=cfg.K, q_hi=cfg.q_hi, quanta=cfg.quanta, beta=cfg.beta,
                max_batch=cfg.max_batch, kv_budget=cfg.kv_budget, block_tokens=cfg.block_tokens,
                max_calls=kw.pop("max_calls", 1 << 14), max_programs=kw.pop("max_programs", 1 << 12),
                token_threshold=cfg.token_threshold)
    args.update(kw)
    return Scheduler(**args)


def oracle_records(tr, cfg):
    cfg.block_bytes = 1  # swap ledger in blocks
    log, m = simulate(tr, cfg, check_formulations=False)
    return [(r["t"], r["batch"], r["admit"], r["preempt"], r["swap_out"], r["swap_in"], r["kv_blocks"])
            for r in log if r["batch"] or r["preempt"]], m


def gpu_records(tr, cfg, fused=False, **kw):
    from paper_2502_13965_b200 import TraceDriver
    s = make_sched(cfg, **kw)
    d = TraceDriver(tr, s)
    log = d.run(fused=fused)
    s.close()
    return [(r["t"], r["batch"], r["admit"], r["preempt"], r["swap_out_blocks"], r["swap_in_blocks"],
             r["kv_blocks"]) for r in log if r["batch"] or r["preempt"]]


def assert_same(got, want):
    assert len(got) == len(want), f"{len(got)} vs {len(want)} steps"
    for g, w in zip(got, want):
        assert g == w, f"step {w[0]}: gpu {g} != oracle {w}"


@pytest.mark.parametrize("policy", [FCFS, MLFQ, PLAS, ATLAS])
def test_fig2(policy):
    tr = fig2()
    want, m = oracle_records(tr, fig2_config(policy))
    assert m["total_wait"] == {FCFS: 18, MLFQ: 18, PLAS: 12, ATLAS: 12}[policy]
    assert_same(gpu_records(tr, fig2_config(policy)), want)


@pytest.mark.parametrize("policy", [PLAS, ATLAS])
def test_atlas_dag_fixture(policy):
    tr = atlas_dag_fixture()
    cfg = Config(policy=policy, K=3, q_hi=(2, 6), quanta=(2, 4, None), max_batch=2)
    want, _ = oracle_records(tr, cfg)
    assert_same(gpu_records(tr, Config(policy=policy, K=3, q_hi=(2, 6), quanta=(2, 4, None), max_batch=2)), want)


LADDERS = [dict(K=1, q_hi=(), quanta=(None,)), dict(K=2, q_hi=(1,), quanta=(1, None)),
           dict(K=3, q_hi=(2, 5), quanta=(1, 2, None)), dict(K=4, q_hi=(1, 3, 6), quanta=(2, 1, 3, 2))]
BETAS = [(1, 0), (2, 1), (1, 2), (5, 3)]
BUDGETS = [None, 8, 12]


def tiny_cfg(i, policy):
    return Config(policy=policy, max_batch=1 + i % 3, kv_budget=BUDGETS[(i // 3) % 3],
                  beta=BETAS[(i // 9) % 4], block_tokens=4, **LADDERS[i % 4])


@pytest.mark.parametrize("seed", range(200))
def test_random_tiny(seed):
    tr = random_tiny(seed)
    for p, policy in enumerate((FCFS, MLFQ, PLAS, ATLAS)):
        cfg = tiny_cfg(seed * 4 + p, policy)
        try:
            want, _ = oracle_records(tr, cfg)
        except CapacityError:
            # a call outgrows P while decoding: the CUDA path must fail with E_NOMEM too
            from paper_2502_13965_b200 import AutxError
            with pytest.raises(AutxError) as e:
                gpu_records(tr, tiny_cfg(seed * 4 + p, policy))
            assert e.value.code == 4
            continue
        except ValueError:
            continue  # a call's initial kvb exceeds P: the ABI rejects it too (tested below)
        assert_same(gpu_records(tr, tiny_cfg(seed * 4 + p, policy)), want)


@pytest.mark.parametrize("seed", [3, 11, 29, 57])
def test_fused_step_entry_point(seed):
    """autx_step (one call per step) reaches the oracle's decisions like the five-call sequence."""
    tr = random_tiny(seed)
    n = 0
    for p, policy in enumerate((FCFS, MLFQ, PLAS, ATLAS)):
        cfg = tiny_cfg(seed * 4 + p, policy)
        try:
            want, _ = oracle_records(tr, cfg)
        except CapacityError:
            continue
        assert_same(gpu_records(tr, tiny_cfg(seed * 4 + p, policy), fused=True), want)
        n += 1
    assert n > 0


@pytest.mark.parametrize("seed", range(24))
def test_steps_across_2_31(seed):
    """Traces whose steps cross 2^31: the dense pass leaves its 32-bit fast path for the exact
    128-bit anti-starvation comparison (R25: u32 steps, u64 products) and must still agree."""
    import dataclasses
    off = (1 << 31) - 2  # most traces cross 2^31 within their first steps
    tr = random_tiny(seed)
    tr = dataclasses.replace(tr, prog_arrival=tr.prog_arrival + off)
    policy = (FCFS, MLFQ, PLAS, ATLAS)[seed % 4]
    cfg = tiny_cfg(seed * 4 + 2, policy)
    cfg.kv_budget = None
    cfg.beta = [(2, 1), (1, 2), (5, 3)][seed % 3]
    cfg.block_bytes = 1
    log, _ = simulate(tr, cfg, max_steps=100_000, start=off)
    want = [(r["t"], r["batch"], r["admit"], r["preempt"], r["swap_out"], r["swap_in"], r["kv_blocks"])
            for r in log if r["batch"] or r["preempt"]]
    assert want
    assert_same(gpu_records(tr, cfg), want)


def normalize_oracle_state(eng: Engine, cfg: Config):
    """Oracle state after phase 7 in table order, with the next step's demotion (phase 3)
    applied: the CUDA path demotes eagerly at the end of the step."""
    rows = []
    for c in sorted(eng.calls.values(), key=lambda c: c.seq):
        q, qt = c.q, c.quanta
        if qt is not None and qt <= 0:
            q = min(q + 1, cfg.K - 1)
            qt = cfg.quanta[q]
        flags = (1 if c.running else 0) | (2 if c.resident else 0) | (4 if (not c.resident and c.exec > 0) else 0)
        rows.append((c.cid, q, 0xFFFFFFFF if qt is None else qt, c.wait, c.mtime, c.exec, c.totwait,
                     c.inh, c.input_tokens, c.arr, flags))
    return rows


@pytest.mark.parametrize("seed", range(40))
def test_state_after_every_step(seed):
    """Full per-call state (queue, quantum, wait, model time, exec, total wait, inherited
    service, flags) and program table equal the oracle's after every step."""
    state_parity(seed, (FCFS, MLFQ, PLAS, ATLAS)[seed % 4])


@pytest.mark.parametrize("seed", range(30))
def test_state_after_every_step_eq2(seed):
    """Exact Eq. 2 ATLAS: every call's inherited priority is max over its parents of
    p + t, checked in the full state dump after every step."""
    state_parity(seed, ATLAS_EQ2, max_calls=7)


def state_parity(seed, policy, max_calls=5):
    from paper_2502_13965_b200 import TraceDriver
    tr = random_tiny(seed, max_programs=4, max_calls=max_calls)
    cfg = tiny_cfg(seed, policy)
    cfg.kv_budget = None
    eng = Engine(cfg, check_formulations=True)
    wl = Workload(tr)
    s = make_sched(cfg)
    d = TraceDriver(tr, s)
    completed = []
    for t in range(200):
        if wl.finished():
            break
        cids = [int(tr.call_id[c]) for c in completed]
        ended = wl.release(t, completed)
        arr = wl.arrivals(t)
        eng.step(t, cids, arr, wl.parents_of(arr) if policy == ATLAS_EQ2 else None)
        for pid in ended:
            eng.end_program(pid)
        rec_o = eng.prev_batch
        completed = wl.ran(t, rec_o)
        if d.t != t:  # GPU driver skips idle steps
            assert not rec_o and not eng.calls
            continue
        rec = d.step()
        assert rec["batch"] == rec_o
        got = [tuple(int(x) for x in r) for r in s.dump_calls()]
        assert got == normalize_oracle_state(eng, cfg), f"t={t}"
        for pid in eng.table.svc:
            svc, pw = s.program_state(pid)
            assert (svc, pw) == (eng.table.svc[pid], eng.table.pwait[pid])
    s.close()


@pytest.mark.parametrize("policy,kv", [(PLAS, None), (PLAS, 2400), (ATLAS, 3000), (MLFQ, 2400)])
def test_chatbot_slice(policy, kv):
    """ShareGPT-shaped chains, SPEC ladder, beta = 2, BS = 32, a binding KV
    budget: many preemptions, promotions and swaps."""
    tr = chatbot(300)
    cfg = spec_ladder_config(policy, max_batch=32, kv_budget=kv)
    want, _ = oracle_records(tr, cfg)
    assert_same(gpu_records(tr, spec_ladder_config(policy, max_batch=32, kv_budget=kv)), want)


def test_react_slice():
    tr = react(400)
    cfg = spec_ladder_config(PLAS, max_batch=64, kv_budget=4000)
    want, _ = oracle_records(tr, cfg)
    assert_same(gpu_records(tr, spec_ladder_config(PLAS, max_batch=64, kv_budget=4000)), want)


def test_mcts_mapreduce_slice_multi_tile():
    """DAG programs (fork/join) at a size spanning many 1024-row scan tiles with a ragged tail."""
    tr = mcts_mapreduce(120)
    assert tr.n_calls > 5000
    cfg = spec_ladder_config(ATLAS, max_batch=256, kv_budget=20000)
    want, _ = oracle_records(tr, cfg)
    assert_same(gpu_records(tr, spec_ladder_config(ATLAS, max_batch=256, kv_budget=20000),
                            max_calls=1 << 16), want)


@pytest.mark.parametrize("seed", range(100))
def test_random_tiny_eq2(seed):
    """Exact Eq. 2 mode on random DAGs (forks, 2-parent joins, interrupt delays), decisions."""
    tr = random_tiny(seed, max_calls=6)
    cfg = tiny_cfg(seed * 4 + 3, ATLAS_EQ2)
    try:
        want, _ = oracle_records(tr, cfg)
    except (CapacityError, ValueError):
        return  # capacity cases are covered by test_random_tiny
    assert_same(gpu_records(tr, tiny_cfg(seed * 4 + 3, ATLAS_EQ2)), want)


def test_eq2_golden_fork():
    """tests/golden/eq2_fork.json: Eq. 2 gives c3 priority 5 where the scalar gives 9; with a
    queue bound between them the two modes place c3 in different queues."""
    import json
    import os
    from autx_workload import dag_trace
    from paper_2502_13965_b200 import TraceDriver
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "eq2_fork.json")))
    tr = dag_trace("eq2_fork", [g["trace"]], [0])
    for pol, key in ((ATLAS_EQ2, "inh_eq2"), (ATLAS, "inh_atlas")):
        cfg = Config(policy=pol, K=2, q_hi=(6,), quanta=(None, None), max_batch=4)
        s = make_sched(cfg)
        d = TraceDriver(tr, s)
        seen = {}
        while d.skip_idle():
            d.step()
            for r in s.dump_calls():
                seen.setdefault(str(int(r["call_id"]) & 0xFFFF), int(r["inh"]))
        s.close()
        assert seen == g[key], pol


@pytest.mark.parametrize("frac", [0.0, 0.5, 1.0])
def test_eq2_mcts_mapreduce_slice(frac):
    """MCTS and map-reduce DAGs in Eq. 2 mode over many scan tiles, binding KV budget."""
    tr = mcts_mapreduce(60, seed=11, frac_mcts=frac)
    cfg = spec_ladder_config(ATLAS_EQ2, max_batch=128, kv_budget=12000)
    want, _ = oracle_records(tr, cfg)
    assert_same(gpu_records(tr, spec_ladder_config(ATLAS_EQ2, max_batch=128, kv_budget=12000),
                            max_calls=1 << 16), want)


def test_eq2_with_kv_allocator():
    """Exact Eq. 2 with the GPU block allocator on (the full finalize path: swap plan, block tables)
    and a binding budget: decisions and swap blocks equal the oracle's."""
    tr = mcts_mapreduce(30, seed=5, frac_mcts=0.5)
    P = 6000
    want, _ = oracle_records(tr, spec_ladder_config(ATLAS_EQ2, max_batch=64, kv_budget=P))
    got = gpu_records(tr, spec_ladder_config(ATLAS_EQ2, max_batch=64, kv_budget=P), max_calls=1 << 16,
                      n_gpu_blocks=P, max_blocks_per_call=4096, host_pages=1 << 16)
    assert_same(got, want)


def test_eq2_protocol_errors():
    from paper_2502_13965_b200 import Scheduler, AutxError, CALL_DESC
    with pytest.raises(AutxError):
        Scheduler(policy="atlas_eq2", max_batch=2, max_calls=64, max_programs=8, rank=0, nranks=2)
    s = Scheduler(policy="atlas_eq2", K=1, quanta=(None,), max_batch=2, max_calls=64, max_programs=8)

    def desc(cids, pids, t):
        d = np.zeros(len(cids), CALL_DESC)
        d["call_id"], d["program_id"], d["arrival_step"] = cids, pids, t
        return d
    s.register_dag(desc([1, 2], [7, 8], 0), [0, 0, 0], [])
    s.sched_step(0)
    for cid, code in ((99, 2), (1, 5)):          # unknown parent; parent still active
        with pytest.raises(AutxError) as e:
            s.register_dag(desc([3], [7], 1), [0, 1], [cid])
        assert e.value.code == code
    s.complete([1, 2])
    with pytest.raises(AutxError) as e:          # parent of another program
        s.register_dag(desc([3], [7], 1), [0, 1], [2])
    assert e.value.code == 1
    s.register_dag(desc([3], [7], 1), [0, 1], [1])   # p = 0 + 1
    s.sched_step(1)
    assert [int(r["inh"]) for r in s.dump_calls()] == [1]
    s.close()
    p = Scheduler(policy="plas", max_batch=2, max_calls=64, max_programs=8)
    with pytest.raises(AutxError) as e:
        p.register_dag(desc([1], [7], 0), [0, 0], [])
    assert e.value.code == 1
    p.close()


def test_compaction_preserves_schedule():
    """A call table much smaller than the trace forces stable compaction (G8) many times."""
    tr = chatbot(200)
    cfg = spec_ladder_config(PLAS, max_batch=16, kv_budget=None)
    want, _ = oracle_records(tr, cfg)
    assert_same(gpu_records(tr, spec_ladder_config(PLAS, max_batch=16), max_calls=400), want)


@pytest.mark.parametrize("policy,kv", [(PLAS, 2400), (ATLAS, None), (ATLAS_EQ2, 3000)])
def test_device_compaction_with_kv_allocator(policy, kv):
    """Device-side G8 compaction (double-buffered table, k_live_count / k_compact /
    k_remap_prev) under the KV block allocator (resident slots and host pages move with their
    rows) and exact Eq. 2 (lineage by call id): lists and ledgers equal the oracle's, and the
    table really was compacted many times."""
    from paper_2502_13965_b200 import TraceDriver
    tr = mcts_mapreduce(12) if policy == ATLAS_EQ2 else chatbot(200)
    mk = lambda: spec_ladder_config(policy, max_batch=16, kv_budget=kv)
    want, _ = oracle_records(tr, mk())
    extra = dict(n_gpu_blocks=kv, max_blocks_per_call=4096, host_pages=1 << 14) if kv else {}
    s = make_sched(mk(), max_calls=650 if policy == ATLAS_EQ2 else 400, **extra)
    log = TraceDriver(tr, s).run()
    n, us = s.compaction_stats()
    s.close()
    got = [(r["t"], r["batch"], r["admit"], r["preempt"], r["swap_out_blocks"], r["swap_in_blocks"],
            r["kv_blocks"]) for r in log if r["batch"] or r["preempt"]]
    assert_same(got, want)
    assert n >= (1 if policy == ATLAS_EQ2 else 3)


def test_protocol_errors():
    from paper_2502_13965_b200 import Scheduler, AutxError, CALL_DESC
    s = Scheduler(policy="plas", K=2, q_hi=(1,), quanta=(1, None), max_batch=1, kv_budget=4,
                  block_tokens=4, max_calls=64, max_programs=8)
    d = np.zeros(2, CALL_DESC)
    d["call_id"] = [5, 4]
    d["program_id"] = [1, 1]
    with pytest.raises(AutxError) as e:        # not canonical
        s.register(d)
    assert e.value.code == 1
    d["call_id"] = [4, 5]
    d["input_tokens"] = [0, 100]               # kvb(100) = 26 > P = 4
    with pytest.raises(AutxError) as e:
        s.register(d)
    assert e.value.code == 1
    d["input_tokens"] = [0, 0]
    s.register(d)
    s.sched_step(0)
    b, _, _ = s.lists()
    assert list(b) == [4]
    with pytest.raises(AutxError) as e:        # call 5 did not run
        s.complete([5])
    assert e.value.code == 5
    with pytest.raises(AutxError) as e:        # unknown
        s.complete([99])
    assert e.value.code == 2
    with pytest.raises(AutxError) as e:        # active calls: end_program refused
        s.end_program(1)
    assert e.value.code == 5
    with pytest.raises(AutxError) as e:        # step must increase
        s.sched_step(0)
    assert e.value.code == 5
    s.complete([4])
    s.sched_step(1)
    s.close()


@pytest.mark.parametrize("mode,pool", [(0, 1), (2, 1), (1, 1), (0, 2), (2, 2)])
def test_kv_swap_round_trip_bytes(mode, pool):
    """Swap-out then swap-in through the C ABI moves exactly the oracle's blocks and restores
    every preempted call's KV contents byte for byte, possibly into other GPU blocks.  Modes:
    0 SM-driven copy, 2 staged DMA (the paper's scheme), 1 per-chunk cudaMemcpyAsync (vLLM).
    pool = 2: a block pool twice the budget, where swap-ins take blocks freed by earlier steps and
    the two directions run at the same time (full duplex) on most steps."""
    import torch
    from paper_2502_13965_b200 import TraceDriver
    tr = chatbot(120)
    L, chunk = 2, 1024
    P = 2400
    nblk = pool * P
    cfg = spec_ladder_config(PLAS, max_batch=16, kv_budget=P)
    want, _ = oracle_records(tr, cfg)
    s = make_sched(spec_ladder_config(PLAS, max_batch=16, kv_budget=P), n_gpu_blocks=nblk,
                   max_blocks_per_call=4096, host_pages=1 << 14)
    kpools = [torch.zeros(nblk, chunk // 4, dtype=torch.int32, device="cuda") for _ in range(L)]
    vpools = [torch.zeros(nblk, chunk // 4, dtype=torch.int32, device="cuda") for _ in range(L)]
    host = torch.zeros((1 << 14) * L * 2 * chunk // 4, dtype=torch.int32).pin_memory()
    d = TraceDriver(tr, s)
    written = {}   # call id -> number of leading blocks whose contents the "engine" wrote
    moved_out = moved_in = 0
    got = []
    duplex = both = 0

    def pat(cid, j, l, kv):
        return (cid * 1000003 + j * 101 + l * 7 + kv) & 0x7FFFFFFF

    while not d.finished():
        if len(d.pending) == 0 and s.num_active() == 0 and d.t not in d.ready:
            d.t = min(d.ready)
        rec = d.step()
        st = s.kv_swap([p.data_ptr() for p in kpools], [p.data_ptr() for p in vpools], chunk,
                       host.data_ptr(), host.numel() * 4, mode)
        assert st.bytes_d2h == rec["swap_out_blocks"] * L * 2 * chunk
        assert st.bytes_h2d == rec["swap_in_blocks"] * L * 2 * chunk
        moved_out += st.bytes_d2h
        moved_in += st.bytes_h2d
        duplex += st.duplex
        both += st.bytes_d2h > 0 and st.bytes_h2d > 0
        offs, blks = s.block_table_host()
        chk_idx, chk_val, new_idx, new_val = [], [], [], []
        for i, cid in enumerate(rec["batch"]):
            mine = blks[offs[i]:offs[i + 1]]
            w = written.get(cid, 0)
            assert len(mine) >= w
            for j in range(len(mine)):
                (chk_idx if j < w else new_idx).append(int(mine[j]))
                (chk_val if j < w else new_val).append((cid, j))
            written[cid] = len(mine)
        for l in range(L):
            for kv, pools in ((0, kpools), (1, vpools)):
                if chk_idx:
                    idx = torch.tensor(chk_idx, device="cuda", dtype=torch.long)
                    exp = torch.tensor([pat(c, j, l, kv) for c, j in chk_val], device="cuda", dtype=torch.int32)
                    assert bool((pools[l][idx] == exp[:, None]).all()), f"KV corrupted at t={rec['t']}"
                if new_idx:
                    idx = torch.tensor(new_idx, device="cuda", dtype=torch.long)
                    val = torch.tensor([pat(c, j, l, kv) for c, j in new_val], device="cuda", dtype=torch.int32)
                    pools[l][idx] = val[:, None].expand(-1, chunk // 4)
        got.append((rec["t"], rec["batch"], rec["admit"], rec["preempt"], rec["swap_out_blocks"],
                    rec["swap_in_blocks"], rec["kv_blocks"]))
    got = [g for g in got if g[1] or g[3]]
    assert_same(got, want)
    assert moved_out > 0 and moved_in > 0
    if pool == 2 and mode != 1:
        assert both > 0 and duplex >= both // 2, (duplex, both)
    s.close()


@pytest.mark.parametrize("seed", range(60))
def test_radix_order_tiny(seed):
    """AUTX_ORDER_RADIX (full LSD radix sort of packed keys) against the oracle."""
    from paper_2502_13965_b200 import ORDER_RADIX
    tr = random_tiny(seed)
    policy = (FCFS, MLFQ, PLAS, ATLAS)[seed % 4]
    cfg = tiny_cfg(seed * 3, policy)
    try:
        want, _ = oracle_records(tr, cfg)
    except ValueError:
        return
    assert_same(gpu_records(tr, tiny_cfg(seed * 3, policy), order_mode=ORDER_RADIX), want)


@pytest.mark.parametrize("policy", [PLAS, ATLAS])
def test_radix_order_multi_tile(policy):
    """Radix path over several 4096-key tiles with a ragged tail and a binding KV budget."""
    from paper_2502_13965_b200 import ORDER_RADIX
    tr = mcts_mapreduce(150) if policy == ATLAS else chatbot(1500)
    cfg = spec_ladder_config(policy, max_batch=256, kv_budget=20000)
    want, _ = oracle_records(tr, cfg)
    assert_same(gpu_records(tr, spec_ladder_config(policy, max_batch=256, kv_budget=20000),
                            order_mode=ORDER_RADIX, max_calls=1 << 16), want)


@pytest.mark.parametrize("policy,steps", [(ATLAS, 30), (ATLAS_EQ2, 12)])
def test_full_size_1m_burst_first_steps(policy, steps):
    """BASELINE configs[3] at full size, in bench.py's launch configuration (select mode, graph
    replay, ATLAS, SPEC ladder, beta 2, BS 1024, P 32768): the first 30 steps of the 1M-call burst
    (registration of every call, then steady steps with completions and arrivals) decide exactly
    what the oracle decides, list for list."""
    from autx_workload import burst_mcts_mapreduce, BASE_SEED, CONFIG_INDEX
    from paper_2502_13965_b200 import TraceDriver
    tr = burst_mcts_mapreduce(1_000_000, seed=BASE_SEED + CONFIG_INDEX["mcts"])
    cfg = spec_ladder_config(policy, max_batch=1024, kv_budget=32768)
    eng = Engine(cfg, check_formulations=False)
    wl = Workload(tr)
    s = make_sched(spec_ladder_config(policy, max_batch=1024, kv_budget=32768),
                   max_calls=1_300_000, max_programs=tr.n_programs + 1024)
    d = TraceDriver(tr, s)
    completed = []
    for t in range(steps):
        cids = [int(tr.call_id[c]) for c in completed]
        ended = wl.release(t, completed)
        arr = wl.arrivals(t)
        rec_o = eng.step(t, cids, arr, wl.parents_of(arr) if policy == ATLAS_EQ2 else None)
        for pid in ended:
            eng.end_program(pid)
        completed = wl.ran(t, rec_o["batch"])
        rec = d.step()
        assert rec["n_active"] == rec_o["n_active"] > 900_000
        assert (rec["batch"], rec["admit"], rec["preempt"]) == (rec_o["batch"], rec_o["admit"], rec_o["preempt"]), t
    s.close()


@pytest.mark.parametrize("workload", ["chatbot", "react"])
def test_full_size_chatbot_react_first_steps(workload):
    """BASELINE configs[1] (10k ShareGPT-shaped programs, BS 256) and configs[2] (100k BFCL-shaped
    programs, BS 256) at full size with the bench's PLAS configuration and KV budgets: 40 steps of
    lists equal to the oracle's."""
    from autx_workload import chatbot, react
    from paper_2502_13965_b200 import TraceDriver
    tr, P = (chatbot(10_000), 6000) if workload == "chatbot" else (react(100_000), 8000)
    cfg = spec_ladder_config(PLAS, max_batch=256, kv_budget=P)
    eng = Engine(cfg, check_formulations=False)
    wl = Workload(tr)
    s = make_sched(spec_ladder_config(PLAS, max_batch=256, kv_budget=P), max_calls=tr.n_programs + 4096,
                   max_programs=tr.n_programs + 1024)
    d = TraceDriver(tr, s)
    completed = []
    for t in range(40):
        cids = [int(tr.call_id[c]) for c in completed]
        ended = wl.release(t, completed)
        rec_o = eng.step(t, cids, wl.arrivals(t))
        for pid in ended:
            eng.end_program(pid)
        completed = wl.ran(t, rec_o["batch"])
        if d.t != t:  # the driver skips steps with nothing active
            assert not rec_o["batch"]
            continue
        rec = d.step()
        assert rec["n_active"] == rec_o["n_active"]
        assert (rec["batch"], rec["admit"], rec["preempt"]) == (rec_o["batch"], rec_o["admit"], rec_o["preempt"]), t
    s.close()


@pytest.mark.parametrize("bs,P,X,kv", [(2048, None, 0, False), (1536, 60000, 0, True), (1024, 60000, 1024, True),
                                        (2000, None, 0, False)])
def test_large_batch_saturated(bs, P, X, kv):
    """Resident sets above 1024 (BS up to the 2048 cap, or BS + X over-provisioned): the finalize's
    1024-thread variant and k_rank's shared memory at 2 x 2048 keys, with more active calls than the
    resident set can take (saturated), 60 steps side by side with the oracle, lists and ledgers."""
    from paper_2502_13965_b200 import TraceDriver
    tr = chatbot(2600)
    mk = lambda: Config(**{**spec_ladder_config(PLAS, max_batch=bs, kv_budget=P).__dict__, "overprovision": X,
                           "block_bytes": 1})
    eng = Engine(mk(), check_formulations=False)
    wl = Workload(tr)
    extra = dict(n_gpu_blocks=P, max_blocks_per_call=4096, host_pages=1 << 18) if kv else {}
    s = make_sched(mk(), max_calls=tr.n_calls + 4096, max_programs=tr.n_programs + 1024, overprovision=X, **extra)
    d = TraceDriver(tr, s)
    completed, saturated = [], 0
    for t in range(60):
        cids = [int(tr.call_id[c]) for c in completed]
        ended = wl.release(t, completed)
        rec_o = eng.step(t, cids, wl.arrivals(t))
        for pid in ended:
            eng.end_program(pid)
        completed = wl.ran(t, rec_o["batch"])
        rec = d.step()
        saturated += rec["n_active"] > bs + X
        assert (rec["batch"], rec.get("standby", []), rec["admit"], rec["preempt"]) == \
            (rec_o["batch"], rec_o.get("standby", []), rec_o["admit"], rec_o["preempt"]), t
        assert (rec["swap_out_blocks"], rec["swap_in_blocks"], rec["kv_blocks"]) == \
            (rec_o["swap_out"], rec_o["swap_in"], rec_o["kv_blocks"]), t
    assert saturated >= 50
    s.close()


def oracle_from_snapshot(s, tr, cfg, d):
    """The oracle's engine state rebuilt from a GPU snapshot (SURVEY §8(d) timing protocol step
    1): every active call's state from autx_dump_calls (table order = registration order), the
    process table of every live program from autx_program_state, the previous batch in order."""
    from oracle.autellix import Call
    st = s.dump_calls()
    eng = Engine(cfg, check_formulations=False)
    for i, r in enumerate(st):
        cid = int(r["call_id"])
        p = cid >> 16
        qt = int(r["quanta"])
        tok, ex = int(r["input_tokens"]), int(r["exec"])
        eng.calls[cid] = Call(cid=cid, pid=int(tr.prog_id[p]), arr=int(r["arrival_step"]),
                              parr=int(tr.prog_arrival[p]), seq=i, input_tokens=tok, inh=int(r["inh"]),
                              q=int(r["q"]), quanta=None if qt == 0xFFFFFFFF else qt, wait=int(r["wait"]),
                              mtime=int(r["mtime"]), exec=ex, totwait=int(r["totwait"]),
                              running=bool(r["flags"] & 1), resident=bool(r["flags"] & 2),
                              held=-(-(tok + ex) // cfg.block_tokens) if ex else 0)
    eng.next_seq = len(st)
    for p in np.nonzero(d.calls_left > 0)[0]:
        pid = int(tr.prog_id[p])
        svc, pw = s.program_state(pid)
        eng.table.svc[pid], eng.table.pwait[pid] = svc, pw
        eng.table.last_arrival[pid], eng.table.last_completion[pid] = 0, None
    eng.prev_batch = list(d.log[-1]["batch"])
    return eng


@pytest.mark.parametrize("policy", [ATLAS, PLAS])
def test_full_size_1m_snapshot_after_10k_steps(policy):
    """BASELINE configs[3] at full size in the bench's state: the GPU runs the 1M-call burst for
    10,000 steps (the bench's fast-forward), the oracle is rebuilt from the GPU's snapshot, and
    the two then run 10 steps side by side with the same completions and arrivals: lists equal
    every step, and the full per-call state and the touched programs' table rows equal at the
    end (the transition function at full scale)."""
    from autx_workload import burst_mcts_mapreduce, BASE_SEED, CONFIG_INDEX
    from paper_2502_13965_b200 import TraceDriver
    tr = burst_mcts_mapreduce(1_000_000, seed=BASE_SEED + CONFIG_INDEX["mcts"])
    cfg = spec_ladder_config(policy, max_batch=1024, kv_budget=32768)
    s = make_sched(spec_ladder_config(policy, max_batch=1024, kv_budget=32768),
                   max_calls=1_300_000, max_programs=tr.n_programs + 1024)
    d = TraceDriver(tr, s, log_lists=False)
    for _ in range(10_000):
        d.step()
    d.log_lists = True  # the previous batch, in order, for the snapshot
    d.step()
    eng = oracle_from_snapshot(s, tr, cfg, d)
    assert len(eng.calls) > 800_000
    touched = set()
    for _ in range(10):
        t = d.t
        cids = [int(x) for x in tr.call_id[d.pending]]
        touched.update(int(tr.prog_id[int(c) >> 16]) for c in cids)
        left = d.calls_left.copy()
        rec = d.step()
        arr = [(int(tr.call_id[c]), int(tr.prog_id[tr.call_prog[c]]), t, int(tr.prog_arrival[tr.call_prog[c]]),
                int(tr.input_tokens[c])) for c in d.arr_idx]
        rec_o = eng.step(t, cids, arr)
        for p in np.nonzero((left > 0) & (d.calls_left == 0))[0]:
            eng.end_program(int(tr.prog_id[p]))
        assert rec["n_active"] == rec_o["n_active"]
        assert (rec["batch"], rec["admit"], rec["preempt"]) == (rec_o["batch"], rec_o["admit"], rec_o["preempt"]), t
    got = [tuple(int(x) for x in r) for r in s.dump_calls()]
    assert got == normalize_oracle_state(eng, cfg)
    for pid in sorted(touched):
        if pid in eng.table.svc:
            assert s.program_state(pid) == (eng.table.svc[pid], eng.table.pwait[pid]), pid
    s.close()


def test_program_latency_of_gpu_schedules():
    """SURVEY §8(f) item 4 on the CUDA path's decisions: the program-level token latency
     and its tail computed from the GPU decision log equal the oracle's."""
    from oracle.metrics import program_latency, latency_summary
    from paper_2502_13965_b200 import TraceDriver
    tr = chatbot(300)
    cfg = spec_ladder_config(PLAS, max_batch=32, kv_budget=2400)
    olog, _ = simulate(tr, cfg, check_formulations=False)
    s = make_sched(spec_ladder_config(PLAS, max_batch=32, kv_budget=2400))
    glog = TraceDriver(tr, s).run()
    s.close()
    assert program_latency(tr, glog) == program_latency(tr, olog)
    assert latency_summary(program_latency(tr, glog))["p99"] > 0
