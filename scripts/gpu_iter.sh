#!/bin/bash
# One development iteration on a B200: build, a parity subset, the headline bench.
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { tail -20 gpurun_out/r02/build.log; exit 1; }
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "${PYTEST_K:-fig2 or atlas_dag or (random_tiny and 1) or chatbot or state_after or mcts or 1m_burst}" > gpurun_out/r02/iter_pytest.log 2>&1
tail -2 gpurun_out/r02/iter_pytest.log
BENCHES=${BENCHES:-"headline=--no-swap+--no-cpu-baseline+--steps+100"} bash scripts/gpu_bench.sh 2>&1 | grep -v "^== \|api"
