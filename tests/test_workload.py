"""Generator targets: sample means within +-10%
of the paper's per-workload statistics."""
import numpy as np
import pytest

from autx_workload import chatbot, react, mcts_mapreduce, fig2, random_tiny


def close(x, target, tol=0.10):
    return abs(x - target) <= tol * target


def test_sharegpt_stats():
    t = chatbot(10_000)
    t.validate()
    assert close(np.diff(t.first_call).mean(), 6.66)
    assert np.diff(t.first_call).max() <= 80
    assert close(t.decode.mean(), 277) and close(t.prefill.mean(), 256)


def test_bfcl_stats():
    t = react(10_000)
    assert close(np.diff(t.first_call).mean(), 10.75)
    assert close(t.decode.mean(), 34.14) and close(t.prefill.mean(), 735.06)


def test_lats_stats():
    t = mcts_mapreduce(600, frac_mcts=1.0)
    t.validate()
    assert close(np.diff(t.first_call).mean(), 159.7)
    assert close(t.decode.mean(), 72.6) and close(t.prefill.mean(), 467.2)


def test_determinism_and_structure():
    a, b = mcts_mapreduce(50), mcts_mapreduce(50)
    assert np.array_equal(a.decode, b.decode) and np.array_equal(a.par, b.par)
    f = fig2()
    assert [list(f.decode[f.first_call[p]:f.first_call[p + 1]]) for p in range(4)] == \
        [[4, 3, 1, 1], [3, 3, 4], [1, 2], [4]]
    for s in range(20):
        random_tiny(s).validate()


def test_vectorised_dag_generator_structure():
    """The vectorised MCTS/map-reduce generator gives the documented DAG (expands join all
    evaluates of the previous round; reduce joins all maps) and contexts equal to the plain
    longest-token ancestor recursion."""
    from autx_workload.gen import _dag_ctx, MAX_CONTEXT
    t = mcts_mapreduce(200)
    t.validate()
    for p in range(t.n_programs):
        a, b = t.first_call[p], t.first_call[p + 1]
        parents = [[int(x - a) for x in t.parents(c)] for c in range(a, b)]
        ref = _dag_ctx(t.decode[a:b], t.prefill[a:b], parents)
        assert np.array_equal(np.minimum(ref, MAX_CONTEXT), t.input_tokens[a:b])
        if t.meta["is_mcts"][p]:
            I = (b - a) // 10
            for r in range(I):
                for i in range(5):
                    assert parents[10 * r + i] == ([] if r == 0 else list(range(10 * r - 5, 10 * r)))
                    assert parents[10 * r + 5 + i] == [10 * r + i]
        else:
            assert parents[-1] == list(range(b - a - 1)) and all(not x for x in parents[:-1])
