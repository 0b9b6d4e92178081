#!/bin/bash
# ncu of the standalone finalize (radix mode's k_fin: the step kernel's finalize_core alone).
mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu/build.log 2>&1 || { tail -20 gpurun_out/ncu/build.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:k_fin --launch-skip 20 -c 1 \
  -o gpurun_out/ncu/fin python bench.py --steps 3 --warmup 3 --ff 30 --order radix --no-swap --no-cpu-baseline > gpurun_out/ncu/fin.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu/fin.log
