#!/bin/bash
# Short round-end check on one B200: smoke, default bench line, reference arm, ncu launch list,
# and the GPU test suite (no --set full capture; see gpu_final.sh for the full pass).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python -c "import json;d=json.loads(open('gpurun_out/bench_final.json').read().splitlines()[-1]);print('final', d['value'], round(d['ms_per_step']*1e3,2), d['roofline']['frac'], d['roofline'].get('frac_span'), d['e2e']['value'], d['clocks'])" || tail -5 gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 5 --warmup 3 --ff 20 --no-swap --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
