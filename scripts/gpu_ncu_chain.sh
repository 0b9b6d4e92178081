#!/bin/bash
# ncu of one whole step (the five chain kernels, L2 flushed before the step by the bench) in the
# headline configuration: launch list (gpu__time_duration) + --set full of the same five launches.
mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu/build.log 2>&1 || { tail -20 gpurun_out/ncu/build.log; exit 1; }
K='regex:k_prologue|k_scan_tile|k_gather_ss|k_rank|k_finalize'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" \
  --launch-skip ${SKIP:-10005} -c 25 --csv --log-file gpurun_out/ncu/chain_launches.csv \
  python bench.py --steps 5 --warmup 3 --ff ${FF:-2000} --no-swap --no-cpu-baseline > gpurun_out/ncu/chain_list.log 2>&1
echo "list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k "$K" --launch-skip ${SKIP:-10005} -c 5 \
  -o gpurun_out/ncu/chain_full python bench.py --steps 5 --warmup 3 --ff ${FF:-2000} --no-swap --no-cpu-baseline > gpurun_out/ncu/chain_full.log 2>&1
echo "full rc=$?"
