#!/bin/bash
# scan-side region-A emission (tile 0): parity subset, then the headline A/B against AUTX_SCAN_EMIT=0
mkdir -p gpurun_out/emit
python -c "from paper_2502_13965_b200 import _build; _build.build(force=True)" > gpurun_out/emit/build.log 2>&1 || { tail -30 gpurun_out/emit/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_parity_gpu.py -k "fig2 or atlas_dag or random_tiny or chatbot or react or mcts or compaction or full_size or eq2 or large_batch" > gpurun_out/emit/parity.log 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/emit/parity.log)"
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_multistep_gpu.py > gpurun_out/emit/ms.log 2>&1; echo "ms rc=$? $(tail -1 gpurun_out/emit/ms.log)"
for v in 1 0 1 0; do
  AUTX_SCAN_EMIT=$v timeout 600 python bench.py --steps 300 --warmup 5 --no-swap --no-cpu-baseline > gpurun_out/emit/bench_$v.json 2> gpurun_out/emit/bench_$v.err
  echo "emit=$v rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/emit/bench_$v.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1e3,2),'us p50',round(d['step_ms']['p50']*1e3,2), d['value'], d['roofline']['frac'], 'e2e', round(d['e2e']['ms_per_step']*1e3,1), d['chain_us'])")"
done
AUTX_SCAN_EMIT=1 timeout 600 python bench.py --workload churn --steps 200 --warmup 5 --ff 300 --no-swap --no-cpu-baseline > gpurun_out/emit/churn.json 2> gpurun_out/emit/churn.err
echo "churn rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/emit/churn.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1e3,2),'us p50',round(d['step_ms']['p50']*1e3,2), d['chain_us'])")"
