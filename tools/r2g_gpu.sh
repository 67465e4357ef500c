#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/l2pf_ab.py 0,4,8,16,24 5,7,9 > $O/r2g_l2pf_ab.jsonl 2> $O/r2g_l2pf_ab.err; echo "l2pf rc=$?"; cat $O/r2g_l2pf_ab.jsonl; tail -3 $O/r2g_l2pf_ab.err
timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest -p no:cacheprovider -q "tests/test_model_gpu.py::test_linear_vs_torch" > $O/r2g_synccheck_linear.log 2>&1; echo "sync rc=$?"; grep -E "passed|failed|SUMMARY" $O/r2g_synccheck_linear.log | tail -3
