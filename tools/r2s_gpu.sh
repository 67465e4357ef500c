#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gemm_tail_gpu.py tests/test_llama_gpu.py tests/test_model_gpu.py tests/test_tp_gpu.py > $O/r2s_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/r2s_pytest.log
timeout 900 python tools/gemm_schedule_ab.py 5,7,9 > $O/r2s_tail_ab.jsonl 2> $O/r2s_tail_ab.err; echo "ab rc=$?"; cat $O/r2s_tail_ab.jsonl; tail -3 $O/r2s_tail_ab.err
