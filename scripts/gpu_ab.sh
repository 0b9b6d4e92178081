#!/bin/bash
# headline A/B: this tree vs the tree in build/old_$1 (same box, interleaved)
mkdir -p gpurun_out/ab
python -c "from paper_2502_13965_b200 import _build; _build.build(force=True)" > gpurun_out/ab/build.log 2>&1 || exit 1
(cd build/old_$1 && python -c "from paper_2502_13965_b200 import _build; _build.build(force=True)") > gpurun_out/ab/build_old.log 2>&1 || exit 1
for i in 1 2; do
  for t in . build/old_$1; do
    (cd $t && timeout 600 python bench.py --steps 300 --warmup 5 --no-swap --no-cpu-baseline > /tmp/ab.json 2>/dev/null)
    echo "$t $(python -c "import json;d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1e3,2),'us p50',round(d['step_ms']['p50']*1e3,2),'e2e',round(d['e2e']['ms_per_step']*1e3,1), d['chain_us'])")"
  done
done
