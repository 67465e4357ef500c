#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2d_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/r2d_pytest_gpu.log
timeout 600 python tools/wide_probe.py > $O/r2d_wide_probe.jsonl 2> $O/r2d_wide_probe.err; echo "wide rc=$?"; cat $O/r2d_wide_probe.jsonl; tail -3 $O/r2d_wide_probe.err
timeout 300 python tools/tp_latency.py > $O/r2d_tp_latency.jsonl 2> $O/r2d_tp_latency.err; echo "tp rc=$?"; cat $O/r2d_tp_latency.jsonl; tail -3 $O/r2d_tp_latency.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,launch__grid_size \
  --clock-control none -k regex:linear_kernel --csv --log-file $O/r2d_gemm_l2.csv python tools/gemm_l2_probe.py > /dev/null 2>&1; echo "ncu l2 rc=$?"
T="tests/test_vote_gpu.py tests/test_accept_gpu.py tests/test_model_gpu.py::test_linear_vs_torch tests/test_llama_gpu.py::test_gated_silu_linear tests/test_llama_gpu.py::test_gqa_rope_attention tests/test_llama_gpu.py::test_grouped_drafters_equal_separate_models tests/test_gemm_wide_gpu.py"
timeout 900 compute-sanitizer --tool synccheck --print-limit 30 python -m pytest -p no:cacheprovider -q $T > $O/r2d_sanitizer_synccheck.log 2>&1
echo "synccheck rc=$?"; grep -E "passed|failed|SUMMARY" $O/r2d_sanitizer_synccheck.log | tail -3; grep -o "in [a-z_]*\.cu[h]*:[0-9]*" $O/r2d_sanitizer_synccheck.log | sort | uniq -c | head
timeout 900 python bench.py > $O/r2d_bench.json 2> $O/r2d_bench.err; echo "bench rc=$?"; tail -c 2500 $O/r2d_bench.json
du -sh $O
