#!/bin/bash
# round-2 GPU batch 2: full GPU tests on the refactored GEMM library, blocked-weight A/B,
# TP protocol latency, ncu summaries of vote/accept/drafter step, compute-sanitizer logs
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2c_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r2c_pytest_gpu.log
timeout 900 python tools/wblock_probe.py 16,80,112,176 > $O/r2c_wblock.jsonl 2> $O/r2c_wblock.err; echo "wblock rc=$?"; cat $O/r2c_wblock.jsonl
timeout 300 python tools/tp_latency.py > $O/r2c_tp_latency.jsonl 2> $O/r2c_tp_latency.err; echo "tp rc=$?"; cat $O/r2c_tp_latency.jsonl
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/green_probe tools/green_probe.cu -lcuda \
  && timeout 120 /tmp/green_probe > $O/r2c_green.txt 2>&1; echo "green rc=$?"; cat $O/r2c_green.txt
timeout 600 ncu --set full --clock-control none -k regex:"vote|accept" -c 24 -o /tmp/va python tools/ncu_small.py va > /dev/null 2>&1; echo "ncu va rc=$?"
ncu -i /tmp/va.ncu-rep --page details --csv > $O/r2c_ncu_vote_accept_details.csv 2>/dev/null
ncu -i /tmp/va.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size > $O/r2c_ncu_vote_accept_raw.csv 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/r2c_draft_launches.csv python tools/ncu_small.py draft > /dev/null 2>&1; echo "ncu draft list rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"gemv|attention|rmsnorm|linear|argmax|embed" \
  -s 95 -c 95 -o /tmp/draft python tools/ncu_small.py draft > /dev/null 2>&1; echo "ncu draft rc=$?"
ncu -i /tmp/draft.ncu-rep --page details --csv > $O/r2c_ncu_draft_details.csv 2>/dev/null
T="tests/test_vote_gpu.py tests/test_accept_gpu.py tests/test_model_gpu.py::test_linear_vs_torch tests/test_llama_gpu.py::test_gated_silu_linear tests/test_llama_gpu.py::test_gqa_rope_attention tests/test_llama_gpu.py::test_grouped_drafters_equal_separate_models"
for t in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 30 python -m pytest -p no:cacheprovider -q $T > $O/r2c_sanitizer_$t.log 2>&1
  echo "sanitizer $t rc=$?"; grep -E "passed|failed|SUMMARY" $O/r2c_sanitizer_$t.log | tail -4
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 30 python -m pytest -p no:cacheprovider -q tests/test_tp_gpu.py -k "forward_matches or batch_invariant" > $O/r2c_sanitizer_memcheck_tp.log 2>&1
echo "sanitizer memcheck tp rc=$?"; grep -E "passed|failed|SUMMARY" $O/r2c_sanitizer_memcheck_tp.log | tail -3
du -sh $O
