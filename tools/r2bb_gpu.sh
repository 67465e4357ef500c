#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gemm_gated_gpu.py tests/test_llama_gpu.py 2>&1 | tail -3
timeout 600 python tools/gemm_schedule_ab.py 5,7,9 2>&1 | grep -v "^$"
