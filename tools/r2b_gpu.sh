#!/bin/bash
# round-2 GPU evidence batch: green-context probe, ncu of the small kernels, compute-sanitizer, reference arm
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/green_probe tools/green_probe.cu -lcuda \
  && timeout 120 /tmp/green_probe > $O/r2b_green.txt 2>&1; echo "green rc=$?"
timeout 300 python tools/ncu_small.py all; echo "small rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"vote|accept" -c 24 \
  -o $O/r2b_ncu_vote_accept python tools/ncu_small.py va > $O/r2b_ncu_va.log 2>&1; echo "ncu va rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/r2b_draft_launches.csv python tools/ncu_small.py draft > /dev/null 2>&1; echo "ncu draft list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemv|attention|rmsnorm|linear|argmax|embed" \
  -s 95 -c 95 -o $O/r2b_ncu_draft python tools/ncu_small.py draft > $O/r2b_ncu_draft.log 2>&1; echo "ncu draft rc=$?"
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python -m pytest -p no:cacheprovider -q -x \
    tests/test_vote_gpu.py tests/test_accept_gpu.py \
    "tests/test_model_gpu.py::test_linear_vs_torch" "tests/test_llama_gpu.py::test_gated_silu_linear" \
    "tests/test_llama_gpu.py::test_gqa_rope_attention" "tests/test_llama_gpu.py::test_grouped_drafters_equal_separate_models" \
    "tests/test_tp_gpu.py::test_tp_forward_matches_single_gpu" > $O/r2b_sanitizer_$t.log 2>&1
  echo "sanitizer $t rc=$?"; tail -3 $O/r2b_sanitizer_$t.log
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/r2b_ref.json 2> $O/r2b_ref.err; echo "ref rc=$?"
tail -c 1500 $O/r2b_ref.json
