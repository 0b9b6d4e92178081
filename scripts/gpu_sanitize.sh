#!/bin/bash
# compute-sanitizer over a GPU parity subset: memcheck, racecheck, synccheck, initcheck.
# The PDL chain (pre-wait reads), zero-copy host stores and fire-and-forget atomics are covered by
# the subset (Fig. 2, random tiny traces, the KV allocator + swap round trip, a multi-tile slice).
mkdir -p gpurun_out/sanitize
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sanitize/build.log 2>&1 || exit 1
SUB="fig2 or (random_tiny and (3 or 7)) or kv_swap_round_trip_bytes or atlas_dag or mcts_mapreduce_slice_multi_tile or eq2_with_kv"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  [ "$tool" = "initcheck" ] && extra="--track-unused-memory no"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 --target-processes all \
    python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider -k "$SUB" > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize/$tool.log | tail -2 | tr '\n' ' ')"
done
