#!/bin/bash
mkdir -p gpurun_out/radix
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/radix/build.log 2>&1 || { tail -30 gpurun_out/radix/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_parity_gpu.py tests/test_variants_gpu.py -k "radix" > gpurun_out/radix/parity.log 2>&1; echo "radix parity rc=$? $(tail -1 gpurun_out/radix/parity.log)"
timeout 600 python bench.py --order radix --steps 20 --warmup 3 --ff 2000 --no-swap --no-cpu-baseline > gpurun_out/radix/radix.json 2> gpurun_out/radix/radix.err; echo "radix bench rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/radix/radix.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['roofline']['frac'])")"
timeout 600 python bench.py --workload churn --steps 200 --warmup 5 --ff 2000 --no-swap --no-cpu-baseline > gpurun_out/radix/churn.json 2> gpurun_out/radix/churn.err; echo "churn rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/radix/churn.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['state']['compactions'],d['e2e']['ms_per_step'])")"
