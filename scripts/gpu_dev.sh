#!/bin/bash
# Development loop on one B200: rebuild, the headline bench, the ncu launch list (NCU=1), the
# chain timeline (CHAIN=1), then a parity subset (PYTEST_K over PYTEST_FILES).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/d_build.log 2>&1 || { tail -20 gpurun_out/d_build.log; exit 1; }
timeout 600 python bench.py --steps 200 --no-swap --no-cpu-baseline $BENCH_ARGS > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
python -c "import json;d=json.loads(open('gpurun_out/d_bench.json').read().splitlines()[-1]);print('bench', d['value'], round(d['ms_per_step']*1e3,2), d['roofline']['frac'], d.get('chain_us'), d.get('finalize_phases_us'))" || tail -5 gpurun_out/d_bench.err
for e in $AB; do
  env ${e//+/ } timeout 600 python bench.py --steps 200 --no-swap --no-cpu-baseline $BENCH_ARGS > gpurun_out/d_bench_ab.json 2>> gpurun_out/d_bench.err
  python -c "import json;d=json.loads(open('gpurun_out/d_bench_ab.json').read().splitlines()[-1]);print('$e', d['value'], round(d['ms_per_step']*1e3,2), d.get('chain_us'), d.get('finalize_phases_us'))"
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/d_launches.csv python bench.py --steps 5 --warmup 3 --ff 20 --no-swap --no-cpu-baseline > /dev/null 2>&1
  python scripts/ncu_summary.py gpurun_out/d_launches.csv 2>/dev/null | head -12
fi
if [ -n "$CHAIN" ]; then
  AUTX_NVCC_FLAGS=-DAUTX_CHAIN_STAMPS python -c "import __graft_entry__ as g; g.build()" > gpurun_out/chain_build.log 2>&1
  for e in AUTX_DEFAULT=1 $AB; do
    env ${e//+/ } AUTX_BENCH_CHAIN=1 timeout 600 python bench.py --steps 100 --no-swap --no-cpu-baseline $BENCH_ARGS > gpurun_out/chain_$e.json 2>> gpurun_out/chain.err
    python -c "import json;d=json.loads(open('gpurun_out/chain_$e.json').read().splitlines()[-1]);print('$e', round(d['ms_per_step']*1e3,2), d['chain_us'])"
  done
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
fi
if [ -n "$PYTEST_K" ]; then
  timeout ${PYTEST_TIMEOUT:-1200} python -m pytest ${PYTEST_FILES:-tests} -m gpu -x -q -k "$PYTEST_K" > gpurun_out/d_pytest.log 2>&1
  tail -3 gpurun_out/d_pytest.log
fi
