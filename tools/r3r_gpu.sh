#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_attention_tc_gpu.py > $O/r3r_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/r3r_pytest.log
timeout 300 python tools/attn_tc_ab.py "7:500,7:1000,5:2048,5:4096,13:4096" > $O/r3r_attn_tc_ab.jsonl 2>&1; cat $O/r3r_attn_tc_ab.jsonl
