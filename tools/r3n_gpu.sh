#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 2000 python tools/partition_ab.py "verify_hi_layers=0;verify_hi_layers=30;verify_hi_layers=45;verify_hi_layers=60" 6 2 2>&1 | grep -E "rep|Error|error" | tee $O/r3n_hi_ab.jsonl
