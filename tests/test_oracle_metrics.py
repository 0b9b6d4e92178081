"""oracle/metrics.py against hand-derived values: program-level token
latency (footnote 2 P:L362, interrupt delays excluded: reading R33), the Fig. 2
waiting totals recomputed from the decision logs alone, and the clairvoyant SRPT bound of §6.5.3
 on Fig. 2 (total wait 7 = the brute-force optimum)."""
from fractions import Fraction

import pytest

from autx_workload import fig2, dag_trace, chatbot
from oracle.autellix import simulate, fig2_config, spec_ladder_config, Config, FCFS, MLFQ, PLAS
from oracle.metrics import program_latency, latency_summary, simulate_srpt, total_wait, sweep

TOKENS = {"A": 9, "B": 10, "C": 3, "D": 4}            # Fig. 2a decode steps per program


def lat_by_name(tr, log):
    names = tr.meta["names"]
    return {names[p]: Fraction(r, k) for p, (r, k, _) in enumerate(program_latency(tr, log))}


@pytest.mark.parametrize("policy,finish", [(FCFS, dict(A=12, B=14, C=10, D=8)),
                                           (PLAS, dict(A=12, B=14, C=7, D=5))])
def test_fig2_program_latency(policy, finish):
    """Fig. 2 golden schedules: all programs arrive at 0 with no interrupts,
    so token latency = finish / tokens."""
    tr = fig2()
    log, _ = simulate(tr, fig2_config(policy))
    got = lat_by_name(tr, log)
    assert got == {k: Fraction(finish[k], TOKENS[k]) for k in finish}
    assert latency_summary(program_latency(tr, log))["mean"] == pytest.approx(
        float(sum(Fraction(finish[k], TOKENS[k]) for k in finish) / 4))


@pytest.mark.parametrize("policy,wait", [(FCFS, 18), (MLFQ, 18), (PLAS, 12)])
def test_fig2_total_wait_from_logs(policy, wait):
    """The paper's totals recomputed from nothing but the per-step batches."""
    tr = fig2()
    log, _ = simulate(tr, fig2_config(policy))
    assert total_wait(tr, log) == wait


def test_srpt_fig2_reaches_the_optimum():
    """Hand-derived SRPT schedule on Fig. 2 (program remaining decode steps A9 B10 C3 D4 at t=0):
    C and D run first (C finishes at 3, D at 4), then A and B share the batch: A 12, B 14.  Its
    total wait is 7, the brute-force optimum over all schedules (test_oracle_fig2)."""
    tr = fig2()
    log = simulate_srpt(tr, 2)
    # batches in priority order: at t=3 D1 (1 step of D left) before A1 (9 left)
    assert [r["batch"] for r in log[:4]] == [[131072, 196608], [131073, 196608], [131073, 196608], [196608, 0]]
    assert total_wait(tr, log) == 7
    assert lat_by_name(tr, log) == {"A": Fraction(12, 9), "B": Fraction(14, 10), "C": Fraction(3, 3),
                                    "D": Fraction(4, 4)}


def test_multithreaded_latency_uses_the_critical_path():
    """Footnote 2: fork root(2) -> {x(3), y(1)} -> join z(1), BS 2: the program ends at
    2 + 3 + 1 = 6 over 7 tokens."""
    tr = dag_trace("fork", [dict(decode=[2, 3, 1, 1], parents=[[], [0], [0], [1, 2]])], [0])
    log, _ = simulate(tr, Config(policy=PLAS, K=1, quanta=(None,), max_batch=2))
    assert program_latency(tr, log) == [(6, 7, 6 / 7)]


def test_interrupt_delays_are_not_response_time():
    """Reading R33: chain a(1) -> b(2) with a 5-step tool delay before b: b runs at 6-7,
    the program ends at 8, its serving response is 8 - 5 = 3 steps for 3 tokens."""
    tr = dag_trace("tool", [dict(decode=[1, 2], parents=[[], [0]], delay=[0, 5])], [0])
    log, _ = simulate(tr, Config(policy=PLAS, K=1, quanta=(None,), max_batch=1))
    assert program_latency(tr, log) == [(3, 3, 1.0)]


def test_srpt_gap_directional():
    """Fig. 18: in scheduling-only simulation SRPT's mean program token latency
    is at most PLAS's, and PLAS beats FCFS, on loaded ShareGPT-shaped traces (5 seeds)."""
    def tr_of(lam, s):
        return chatbot(60, seed=100 + s, rate=lam)

    pol = {"fcfs": lambda tr: simulate(tr, Config(policy=FCFS, K=1, quanta=(None,), max_batch=8),
                                       check_formulations=False)[0],
           "plas": lambda tr: simulate(tr, spec_ladder_config(PLAS, max_batch=8), check_formulations=False)[0],
           "srpt": lambda tr: simulate_srpt(tr, 8)}
    rows = {(r["rate"], r["policy"]): r for r in sweep(tr_of, [0.05], pol, 8, seeds=range(5))}
    assert rows[(0.05, "srpt")]["mean"] <= rows[(0.05, "plas")]["mean"] < rows[(0.05, "fcfs")]["mean"]
