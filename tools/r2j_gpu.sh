#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_llama_gpu.py tests/test_model_gpu.py tests/test_paged_gpu.py tests/test_engine_gpu.py tests/test_parity_engine_gpu.py > $O/r2j_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r2j_pytest.log
for rep in 1 2; do
for lib in base new; do
  if [ $lib = base ]; then export MS_LIB=$PWD/paper_2402_15678_b200/lib/libminions_base.so; else unset MS_LIB; fi
  for Q in 5 7; do timeout 300 python tools/llama_verify_breakdown.py llama-2-70b $Q 190 16 2>&1 | grep -E "full|attention" | sed "s/^/$lib /"; done
  timeout 300 python tools/draft_breakdown.py 200 16 3 2>&1 | grep attention | sed "s/^/$lib /"
  timeout 300 python tools/draft_step.py 200 16 3 2>&1 | head -1 | sed "s/^/$lib /"
done; done
