#!/bin/bash
# Parity pass on one B200: build, the GPU tests (PYTEST_K subset, default all), smoke.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p_build.log 2>&1 || { tail -20 gpurun_out/p_build.log; exit 1; }
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest ${PYTEST_FILES:-tests} -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/p_pytest.log 2>&1
tail -25 gpurun_out/p_pytest.log
