#!/bin/bash
mkdir -p gpurun_out/compact
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/compact/build.log 2>&1 || { tail -30 gpurun_out/compact/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_parity_gpu.py -k "compaction or protocol or snapshot" > gpurun_out/compact/parity.log 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/compact/parity.log)"
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_multistep_gpu.py -k "compaction or golden" > gpurun_out/compact/ms.log 2>&1; echo "ms rc=$? $(tail -1 gpurun_out/compact/ms.log)"
timeout 600 python bench.py --workload churn --steps 200 --warmup 5 --ff 2000 --no-swap --no-cpu-baseline > gpurun_out/compact/churn.json 2> gpurun_out/compact/churn.err; echo "churn rc=$?"
tail -c 1500 gpurun_out/compact/churn.json
