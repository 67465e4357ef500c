#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_attention_tc_gpu.py > $O/r3b_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/r3b_pytest.log
timeout 300 python tools/attn_tc_ab.py "5:190,7:190,9:190,7:1000,5:4096" > $O/r3b_attn_tc_ab.jsonl 2>&1; cat $O/r3b_attn_tc_ab.jsonl
