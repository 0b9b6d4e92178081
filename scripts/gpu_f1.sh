#!/bin/bash
# f1 (multi-step scheduling, R32) + autx_route GPU tests and a quick regression subset.
mkdir -p gpurun_out/f1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f1/build.log 2>&1 || { tail -30 gpurun_out/f1/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_multistep_gpu.py > gpurun_out/f1/multistep.log 2>&1; echo "multistep rc=$? $(tail -1 gpurun_out/f1/multistep.log)"
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_multi_gpu.py > gpurun_out/f1/multi.log 2>&1; echo "multi rc=$? $(tail -1 gpurun_out/f1/multi.log)"
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_parity_gpu.py -k "fig2 or random_tiny or kv_swap or chatbot_slice or react_slice or compaction or eq2_with_kv or multi_tile" > gpurun_out/f1/parity.log 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/f1/parity.log)"
