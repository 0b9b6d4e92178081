#!/bin/bash
# Round-end measurement pass on one B200: the default bench line (swap + oracle baseline), the
# reference arm, extra configurations, ncu launch list + --set full capture, GPU tests.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)|NUMA" > gpurun_out/lscpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python -c "import json;d=json.loads(open('gpurun_out/bench_final.json').read().splitlines()[-1]);print('final', d['value'], round(d['ms_per_step']*1e3,2), d['roofline'], d.get('swap',{}).get('sm'), d['e2e']['value'])" || tail -5 gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
for cfg in "--policy atlas_eq2" "--workload chatbot" "--workload react" "--order radix --steps 50"; do
  n=$(echo $cfg | tr -d ' -' | cut -c1-20)
  timeout 600 python bench.py --steps 100 --no-swap --no-cpu-baseline $cfg > gpurun_out/bench_$n.json 2> gpurun_out/bench_$n.err
  python -c "import json;d=json.loads(open('gpurun_out/bench_$n.json').read().splitlines()[-1]);print('$n', d['value'], round(d['ms_per_step']*1e3,2))" || tail -3 gpurun_out/bench_$n.err
done
AUTX_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --ff 10 --active 300000 --no-swap --no-cpu-baseline > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; tail -c 200 gpurun_out/bench_gloo2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 5 --warmup 3 --ff 20 --no-swap --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_tile|k_gather_ss|k_rank|k_finalize|k_prologue" -s 50 -c 5 -o gpurun_out/prof_final python bench.py --steps 3 --warmup 3 --ff 20 --no-swap --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
if [ -n "$TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
fi
