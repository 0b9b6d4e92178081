#!/bin/bash
# The driver's round-end GPU tier: full `pytest -m gpu` + smoke at HEAD.
mkdir -p gpurun_out/tests
python -c "from paper_2502_13965_b200 import _build; _build.build(force=True)" > gpurun_out/tests/build.log 2>&1 || { tail -30 gpurun_out/tests/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/tests/pytest_gpu.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/tests/pytest_gpu.log)"
grep -E "^FAILED|^ERROR" gpurun_out/tests/pytest_gpu.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/tests/smoke.log 2>&1; echo "smoke rc=$? $(tail -2 gpurun_out/tests/smoke.log)"
