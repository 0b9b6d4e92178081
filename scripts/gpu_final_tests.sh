#!/bin/bash
# (a) the driver's GPU tier at HEAD: pytest -m gpu + smoke (normal build);
# (b) the device bounds-check build (AUTX_CHECK, the pool refuses compute-sanitizer) with
#     CUDA_LAUNCH_BLOCKING on the parity, multi-step, swap and compaction suites.
mkdir -p gpurun_out/final
python -c "from paper_2502_13965_b200 import _build; _build.build(force=True)" > gpurun_out/final/build.log 2>&1 || { tail -30 gpurun_out/final/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/final/pytest_gpu.log)"; grep -E "^FAILED|^ERROR" gpurun_out/final/pytest_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/final/smoke.log)"
export AUTX_NVCC_FLAGS=-DAUTX_BOUNDS
python -c "from paper_2502_13965_b200 import _build; _build.build(force=True)" > gpurun_out/final/build_bounds.log 2>&1 || exit 1
CUDA_LAUNCH_BLOCKING=1 timeout 2400 python -m pytest -q -p no:cacheprovider tests/test_parity_gpu.py tests/test_multistep_gpu.py \
  -k "not full_size" > gpurun_out/final/bounds_check.log 2>&1
echo "bounds rc=$? $(tail -1 gpurun_out/final/bounds_check.log) checks_failed=$(grep -c 'AUTX_CHECK failed' gpurun_out/final/bounds_check.log)"
unset AUTX_NVCC_FLAGS
python -c "from paper_2502_13965_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
