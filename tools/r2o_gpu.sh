#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for v in 1025 512; do echo "MS_GV8K=$v"; MS_GV8K=$v timeout 300 python tools/draft_breakdown.py 200 16 3 2>&1 | grep -E "qkv|\"o\"|gate_up|down"; MS_GV8K=$v timeout 300 python tools/draft_step.py 200 16 3 2>&1 | head -1; done
