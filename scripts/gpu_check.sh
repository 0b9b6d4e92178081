#!/bin/bash
# Full GPU test pass + smoke, then the compute-sanitizer subset.
mkdir -p gpurun_out/check
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/check/build.log 2>&1 || { tail -20 gpurun_out/check/build.log; exit 1; }
nvidia-smi > gpurun_out/check/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/check/pytest_gpu.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/check/pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check/smoke.log 2>&1; echo "smoke rc=$?"
bash scripts/gpu_sanitize.sh
