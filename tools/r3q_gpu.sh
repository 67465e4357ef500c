#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/wide_verify_probe.py 16,80,112,128 2>&1 | tail -5 | tee $O/r3q_wide_probe.jsonl
