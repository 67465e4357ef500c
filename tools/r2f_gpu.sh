#!/bin/bash
# round-2 GPU batch f: green-context probe, SM-partition A/B, verify breakdown,
# ncu of vote/accept/drafter step, compute-sanitizer logs
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/green_probe tools/green_probe.cu -lcuda \
  && timeout 120 /tmp/green_probe > $O/r2f_green.txt 2>&1; echo "green rc=$?"; cat $O/r2f_green.txt
timeout 1200 python tools/partition_ab.py 0,16,24,32 6 2 > $O/r2f_partition_ab.jsonl 2> $O/r2f_partition_ab.err; echo "partition rc=$?"
cat $O/r2f_partition_ab.jsonl; tail -5 $O/r2f_partition_ab.err
for Q in 5 7 9; do timeout 300 python tools/llama_verify_breakdown.py llama-2-70b $Q 190 16; done > $O/r2f_breakdown.txt 2>&1; echo "breakdown rc=$?"; cat $O/r2f_breakdown.txt | tail -30
timeout 600 ncu --set full --clock-control none -k regex:"vote|accept" -c 24 -o /tmp/va python tools/ncu_small.py va > /dev/null 2>&1; echo "ncu va rc=$?"
ncu -i /tmp/va.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed > $O/r2f_ncu_vote_accept_raw.csv 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/r2f_draft_launches.csv python tools/ncu_small.py draft > /dev/null 2>&1; echo "ncu draft list rc=$?"
T="tests/test_vote_gpu.py tests/test_accept_gpu.py tests/test_model_gpu.py::test_linear_vs_torch tests/test_llama_gpu.py::test_gated_silu_linear tests/test_llama_gpu.py::test_gqa_rope_attention tests/test_llama_gpu.py::test_grouped_drafters_equal_separate_models tests/test_gemm_wide_gpu.py"
for t in racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 30 python -m pytest -p no:cacheprovider -q $T > $O/r2f_sanitizer_$t.log 2>&1
  echo "sanitizer $t rc=$?"; grep -E "passed|failed|SUMMARY" $O/r2f_sanitizer_$t.log | tail -4
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 30 python -m pytest -p no:cacheprovider -q tests/test_tp_gpu.py > $O/r2f_sanitizer_memcheck_tp.log 2>&1
echo "sanitizer memcheck tp rc=$?"; grep -E "passed|failed|SUMMARY" $O/r2f_sanitizer_memcheck_tp.log | tail -3
du -sh $O
