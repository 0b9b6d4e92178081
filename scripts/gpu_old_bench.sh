#!/bin/bash
# The round-1 pipeline (git 23d9084, shipped as build/oldtree.tar) on the same workload state.
mkdir -p /tmp/old && tar -xf build/oldtree.tar -C /tmp/old
cd /tmp/old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python bench.py --steps 100 --warmup 5 --ff ${FF:-10000} --no-swap --no-cpu-baseline > /tmp/old/out.json 2>/tmp/old/err.txt
python - <<'PY'
import json
d = json.loads(open('/tmp/old/out.json').read().splitlines()[-1])
print("old value %.3e ms/step %.2f us e2e %.3e e2e_us %.1f promo %.0f" % (d["value"], d["ms_per_step"] * 1e3, d["e2e"]["value"], d["e2e"]["ms_per_step"] * 1e3, d["promotions_per_step"]))
print("chain", d.get("chain_us"))
PY
