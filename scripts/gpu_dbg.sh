#!/bin/bash
# debug build with device bounds checks (AUTX_CHECK), then the given tests
mkdir -p gpurun_out/dbg
export AUTX_NVCC_FLAGS=-DAUTX_BOUNDS
python -c "from paper_2502_13965_b200 import _build; _build.build(force=True)" > gpurun_out/dbg/build.log 2>&1 || { tail -30 gpurun_out/dbg/build.log; exit 1; }
for k in "$@"; do
  n=$(echo "$k" | tr -c 'a-zA-Z0-9_-' '_')
  CUDA_LAUNCH_BLOCKING=1 AUTX_NO_GRAPH=1 timeout 900 python -m pytest -q -x -s -p no:cacheprovider "$k" > gpurun_out/dbg/$n.log 2>&1
  echo "$k rc=$? $(tail -1 gpurun_out/dbg/$n.log)"; grep -m5 -E "AUTX_CHECK|E  +" gpurun_out/dbg/$n.log
done
