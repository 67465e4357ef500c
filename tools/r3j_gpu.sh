#!/bin/bash
# compute-sanitizer on the tcgen05 attention kernels (racecheck, synccheck, memcheck)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 5 python -m pytest -q -p no:cacheprovider tests/test_attention_tc_gpu.py > $O/r3j_sanitizer_$tool.log 2>&1
  echo "$tool rc=$? :: $(grep -E 'ERROR SUMMARY|passed|failed' $O/r3j_sanitizer_$tool.log | tr '\n' ' ')"
done
