"""GPU parity of the alternative kernel pipelines behind environment switches (read once per
process by the library, hence one subprocess per variant): each must reach the oracle's decisions
exactly, like the default pipeline does in test_parity_gpu.py."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = {
    "dma_out": {"AUTX_DMA_OUT": "1"},            # host lists by one copy instead of zero-copy stores
    "scan_pre0": {"AUTX_SCAN_PRE": "0"},         # scan reads nothing before the PDL wait
    "scan_pre2": {"AUTX_SCAN_PRE": "2"},         # ... prog, base, mtime before the wait
    "no_graph": {"AUTX_NO_GRAPH": "1"},          # the step's kernels as separate launches, not a graph replay
    "finalize_lists": {"AUTX_FINALIZE_LISTS": "1"},  # finalize cuts the batch and writes the lists (not k_rank)
    "rank_narrow": {"AUTX_RANK_NARROW": "1"},    # half a warp per key in k_rank whatever the candidate count
    "rank_buckets": {"AUTX_RANK_BUCKETS": "1"},  # k_rank's O(BS) bucket ranks instead of the all-pairs count
    "no_gather_prefetch": {"AUTX_GATHER_PREFETCH": "0", "AUTX_FIN_PREV_EARLY": "0"},  # no early reads / prefetches
    "pipeline_ord": {"AUTX_PIPELINE": "ord"},    # no k_rank: the finalize orders the candidates in O(BS)
    "pipeline_sel": {"AUTX_PIPELINE": "sel"},    # no gather, no k_rank: the dense pass emits, the finalize selects
}

# the full-size cases run once, in the default pipeline (test_parity_gpu.py); each variant runs the rest
SUBSET = "(fig2 or atlas_dag or mcts or chatbot or compaction or react or (random_tiny and 7)) and not full_size"


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_parity(name):
    env = dict(os.environ, **VARIANTS[name])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_parity_gpu.py"), "-k", SUBSET],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, f"variant {name} failed:\n{tail}"
    assert " passed" in r.stdout and "failed" not in r.stdout, tail
