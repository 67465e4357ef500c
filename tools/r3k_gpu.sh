#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_attention_tc_gpu.py tests/test_paged_gpu.py tests/test_llama_gpu.py > $O/r3k_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/r3k_pytest.log
timeout 600 compute-sanitizer --tool memcheck python -m pytest -q -p no:cacheprovider tests/test_paged_gpu.py -k bitwise > $O/r3k_memcheck_paged.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $O/r3k_memcheck_paged.log
