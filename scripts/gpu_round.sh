#!/bin/bash
# Round-2 measurement set on one B200 -> gpurun_out/r02/*.json (copied to profiles/r02/ after).
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || { tail -20 gpurun_out/r02/build.log; exit 1; }
nproc > gpurun_out/r02/nproc.txt; lscpu > gpurun_out/r02/lscpu.txt; nvidia-smi > gpurun_out/r02/smi.txt
BENCHES=${BENCHES:-"headline= mixed4m=--workload+mixed4m+--no-swap+--no-cpu-baseline churn=--workload+churn+--ff+300+--no-swap+--no-cpu-baseline betainf=--beta+inf+--no-swap+--no-cpu-baseline chatbot=--workload+chatbot+--no-swap+--no-cpu-baseline react=--workload+react+--no-swap+--no-cpu-baseline eq2=--policy+atlas_eq2+--no-swap+--no-cpu-baseline radix=--order+radix+--steps+30+--no-swap+--no-cpu-baseline"} bash scripts/gpu_bench.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02/reference.json 2> gpurun_out/r02/reference.err
tail -1 gpurun_out/r02/reference.json
