#!/bin/bash
# Bench runs on one B200.  BENCHES: space-separated list of name=args (args with + for spaces);
# default: the headline only.  Results: gpurun_out/${OUT:-r02}/<name>.json (+ .err).
mkdir -p gpurun_out/${OUT:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${OUT:-r02}/build.log 2>&1 || { tail -20 gpurun_out/${OUT:-r02}/build.log; exit 1; }
BENCHES=${BENCHES:-"headline=--no-swap+--no-cpu-baseline"}
for b in $BENCHES; do
  name=${b%%=*}; a=${b#*=}; a=${a//+/ }
  envs=""; args=""
  for tok in $a; do if [[ "$tok" =~ ^[A-Z_]+=.*$ ]]; then envs="$envs $tok"; else args="$args $tok"; fi; done
  timeout ${BENCH_TIMEOUT:-900} env $envs python bench.py $args --json-out gpurun_out/${OUT:-r02}/$name.json > gpurun_out/${OUT:-r02}/$name.out 2> gpurun_out/${OUT:-r02}/$name.err
  echo "== $name rc=$?"
  python - "$name" "${OUT:-r02}" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/{sys.argv[2]}/{n}.json").read())
except Exception as e:
    print("no json:", e); print(open(f"gpurun_out/{sys.argv[2]}/{n}.err").read()[-3000:]); sys.exit(0)
r = d.get("roofline", {})
print(n, "value %.3e" % d["value"], "ms/step %.2f us" % (d["ms_per_step"] * 1e3), "frac", r.get("frac"),
      "e2e %.3e" % d["e2e"]["value"], "e2e us %.1f" % (d["e2e"]["ms_per_step"] * 1e3), "launches/step", d.get("kernels_per_step"))
print("  step_ms", d.get("step_ms"))
print("  chain", d.get("chain_us"), "kern_ev", d.get("kernel_event_ms"))
print("  state", d.get("state"))
print("  api", d["e2e"].get("api_us_per_step"), "clocks", d.get("clocks"))
PY
done
