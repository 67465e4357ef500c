#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python tools/interfere_ab.py 7 5 2>&1 | tail -3 | tee $O/r3o_interfere.jsonl
