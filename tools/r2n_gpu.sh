#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_model_gpu.py tests/test_llama_gpu.py tests/test_engine_gpu.py tests/test_parity_engine_gpu.py tests/test_oracles_gpu.py > $O/r2n_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/r2n_pytest.log
timeout 300 python tools/draft_breakdown.py 200 16 3 2>&1 | tail -8
timeout 300 python tools/draft_step.py 200 16 3 2>&1 | tail -2
