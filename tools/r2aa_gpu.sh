#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_llama_gpu.py tests/test_model_gpu.py tests/test_gemm_wide_gpu.py 2>&1 | tail -3
for M in 16 112 176; do timeout 120 python tools/epi_trace.py $M; done
timeout 300 python tools/epi_probe.py
for Q in 5 7 9; do timeout 300 python tools/llama_verify_breakdown.py llama-2-70b $Q 190 16 2>&1 | grep -E "full|gu"; done
