#!/bin/bash
# ncu --set full of one k_step launch in the headline configuration (L2 flushed before it).
mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu/build.log 2>&1 || { tail -20 gpurun_out/ncu/build.log; exit 1; }
NAME=${NAME:-step}
timeout 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval ${WSI:-5} -k regex:k_step --launch-skip ${SKIP:-300} -c 1 \
  -o gpurun_out/ncu/$NAME python bench.py --steps 5 --warmup 3 --ff ${FF:-400} --no-swap --no-cpu-baseline $BENCH_ARGS > gpurun_out/ncu/$NAME.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu/$NAME.log
ls -la gpurun_out/ncu/
