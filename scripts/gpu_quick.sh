#!/bin/bash
# Quick check on one B200: GPU parity tests, the headline bench, an A/B bench per env setting in
# AB (e.g. AB="AUTX_SELECT_KERNEL=1"), and with NCU=1 a launch list of the default step.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 200 --no-swap --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python -c "import json;d=json.loads(open('gpurun_out/q_bench.json').read().splitlines()[-1]);print('base', d['value'], d['ms_per_step']*1e3, d['breakdown_ms'])"
for e in $AB; do
  env $e timeout 600 python bench.py --steps 200 --no-swap --no-cpu-baseline > gpurun_out/q_bench_ab.json 2>> gpurun_out/q_bench.err
  python -c "import json;d=json.loads(open('gpurun_out/q_bench_ab.json').read().splitlines()[-1]);print('$e', d['value'], d['ms_per_step']*1e3, d['breakdown_ms'])"
done
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1
[ -z "$NOTEST" ] && tail -3 gpurun_out/q_pytest.log
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/q_launches.csv python bench.py --steps 5 --warmup 3 --ff 20 --no-swap --no-cpu-baseline > /dev/null 2>&1
  python scripts/ncu_summary.py gpurun_out/q_launches.csv 2>/dev/null | head -14
fi
