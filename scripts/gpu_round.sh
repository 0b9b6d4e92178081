#!/bin/bash
# Round-2 measurement set on one B200 -> gpurun_out/r02b/*.json (copied to profiles/r02/ after).
mkdir -p gpurun_out/r02b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02b/build.log 2>&1 || { tail -20 gpurun_out/r02b/build.log; exit 1; }
nproc > gpurun_out/r02b/nproc.txt; lscpu > gpurun_out/r02b/lscpu.txt; nvidia-smi > gpurun_out/r02b/smi.txt
OUT=r02b BENCHES=${BENCHES:-"headline= mixed4m=--workload+mixed4m+--no-swap+--no-cpu-baseline churn=--workload+churn+--ff+300+--no-swap+--no-cpu-baseline betainf=--beta+inf+--no-swap+--no-cpu-baseline chatbot=--workload+chatbot+--no-swap+--no-cpu-baseline react=--workload+react+--no-swap+--no-cpu-baseline eq2=--policy+atlas_eq2+--no-swap+--no-cpu-baseline radix=--order+radix+--steps+30+--no-swap+--no-cpu-baseline"} bash scripts/gpu_bench.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02b/reference.json 2> gpurun_out/r02b/reference.err
tail -1 gpurun_out/r02b/reference.json
# whole-step ncu: launch list + one --set full capture (after the benches exited 0 without ncu)
mkdir -p gpurun_out/r02b/ncu
K='regex:k_prologue|k_scan_tile|k_gather_ss|k_rank|k_finalize'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" \
  --launch-skip 10005 -c 25 --csv --log-file gpurun_out/r02b/ncu/chain_launches.csv \
  python bench.py --steps 5 --warmup 3 --ff 2000 --no-swap --no-cpu-baseline > gpurun_out/r02b/ncu/chain_list.log 2>&1
echo "ncu list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k "$K" --launch-skip 10005 -c 5 \
  -o gpurun_out/r02b/ncu/chain_full python bench.py --steps 5 --warmup 3 --ff 2000 --no-swap --no-cpu-baseline > gpurun_out/r02b/ncu/chain_full.log 2>&1
echo "ncu full rc=$?"
