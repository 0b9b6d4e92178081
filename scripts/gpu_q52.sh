timeout 600 python bench.py --steps 200 --no-swap --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python -c "import json;d=json.loads(open('gpurun_out/q_bench.json').read().splitlines()[-1]);print('base', d['value'], d['ms_per_step']*1e3, d['e2e'])"
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_tile" -s 10 -c 1 -o gpurun_out/prof_scan_tile python bench.py --steps 3 --warmup 3 --ff 20 --no-swap --no-cpu-baseline > gpurun_out/ncu_scan.log 2>&1; tail -2 gpurun_out/ncu_scan.log
