#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gemm_sk_gpu.py tests/test_llama_gpu.py tests/test_model_gpu.py > $O/r2m_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/r2m_pytest.log
timeout 900 python tools/sk_ab.py 5,7,9 > $O/r2m_sk_ab.jsonl 2> $O/r2m_sk_ab.err; echo "ab rc=$?"; cat $O/r2m_sk_ab.jsonl; tail -3 $O/r2m_sk_ab.err
