#!/bin/bash
# full-duplex swap: parity + byte round trips, then the bench's swap phase alone
mkdir -p gpurun_out/swap
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/swap/build.log 2>&1 || { tail -30 gpurun_out/swap/build.log; exit 1; }
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_parity_gpu.py -k "kv_swap or eq2_with_kv or react_slice or chatbot_slice" > gpurun_out/swap/parity.log 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/swap/parity.log)"
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_multistep_gpu.py -k "kv" > gpurun_out/swap/ms.log 2>&1; echo "multistep-kv rc=$? $(tail -1 gpurun_out/swap/ms.log)"
timeout 900 python bench.py --steps 5 --warmup 3 --ff 100 --no-cpu-baseline > gpurun_out/swap/bench.json 2> gpurun_out/swap/bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/swap/bench.json
