#!/bin/bash
# One ncu --set full capture (source-correlated) of each step kernel at steady state, plus bench
# lines of extra configurations in EXTRA (e.g. "--policy atlas_eq2").
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_tile|k_gather_ss|k_rank|k_finalize|k_prologue" -s 50 -c 5 -o gpurun_out/prof_${TAG:-n} python bench.py --steps 3 --warmup 3 --ff 20 --no-swap --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
if [ -n "$EXTRA1" ]; then
  timeout 600 python bench.py --steps 200 --no-swap --no-cpu-baseline $EXTRA1 > gpurun_out/n_extra1.json 2> gpurun_out/n_extra1.err
  python -c "import json;d=json.loads(open('gpurun_out/n_extra1.json').read().splitlines()[-1]);print('extra1', d['value'], round(d['ms_per_step']*1e3,2), d['config']['policy'])" || tail -3 gpurun_out/n_extra1.err
fi
