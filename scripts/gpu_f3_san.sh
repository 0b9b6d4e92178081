#!/bin/bash
# f3 router GPU tests + focused sanitizer runs on the Eq. 2 + KV allocator case.
mkdir -p gpurun_out/f3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f3/build.log 2>&1 || exit 1
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_multi_gpu.py > gpurun_out/f3/multi.log 2>&1; echo "multi rc=$? $(tail -1 gpurun_out/f3/multi.log)"
for i in 1 2 3; do
  timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_parity_gpu.py -k eq2_with_kv > gpurun_out/f3/eq2_$i.log 2>&1; echo "eq2 run$i rc=$? $(tail -1 gpurun_out/f3/eq2_$i.log)"
done
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_parity_gpu.py -k eq2_with_kv > gpurun_out/f3/eq2_blocking.log 2>&1; echo "eq2 blocking rc=$? $(tail -1 gpurun_out/f3/eq2_blocking.log)"
AUTX_NO_GRAPH=1 timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_parity_gpu.py -k eq2_with_kv > gpurun_out/f3/eq2_nograph.log 2>&1; echo "eq2 nograph rc=$? $(tail -1 gpurun_out/f3/eq2_nograph.log)"
timeout 900 compute-sanitizer --tool initcheck --print-limit 10 --target-processes all python -m pytest -q -x -p no:cacheprovider tests/test_parity_gpu.py -k eq2_with_kv > gpurun_out/f3/initcheck.log 2>&1; echo "initcheck rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/f3/initcheck.log | tail -1)"
