#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_coresident_gpu.py tests/test_llama_gpu.py tests/test_engine_gpu.py tests/test_parity_engine_gpu.py > $O/r2r_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/r2r_pytest.log
timeout 1200 python tools/partition_ab.py "draft_coresident=1;draft_coresident=0" 6 2 > $O/r2r_co_ab.jsonl 2> $O/r2r_co_ab.err; echo "ab rc=$?"; cat $O/r2r_co_ab.jsonl; tail -3 $O/r2r_co_ab.err
