#!/bin/bash
# Step-chain timeline on one B200: rebuild with -DAUTX_CHAIN_STAMPS, then per-kernel (start, end)
# spans in the PDL-chained step for the default path and each env setting in AB (extra bench
# flags in BENCH_ARGS, e.g. --no-flush).
mkdir -p gpurun_out
AUTX_NVCC_FLAGS=-DAUTX_CHAIN_STAMPS python -c "import __graft_entry__ as g; g.build()" > gpurun_out/chain_build.log 2>&1
for e in AUTX_DEFAULT=1 $AB; do
  env $e AUTX_BENCH_CHAIN=1 timeout 600 python bench.py --steps 100 --no-swap --no-cpu-baseline $BENCH_ARGS > gpurun_out/chain_$e.json 2>> gpurun_out/chain.err
  python -c "import json;d=json.loads(open('gpurun_out/chain_$e.json').read().splitlines()[-1]);print('$e', round(d['ms_per_step']*1e3,2), d['chain_us'])"
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
