#!/bin/bash
export CUDA_LAUNCH_BLOCKING=1 AUTX_NO_GRAPH=1
for t in build/old_c57df7d build/old_dbb35c7 build/old_d420eee .; do
  for hp in 262144; do
    timeout 600 python build/bisect_kv.py $t 1536 $hp 2>&1 | tail -3
  done
done
