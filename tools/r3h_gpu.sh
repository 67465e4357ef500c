#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
for q in 5 7 9; do timeout 600 python tools/verify_attn_ab.py $q 190 2>&1 | tail -1; done | tee $O/r3h_verify_attn_ab.jsonl
