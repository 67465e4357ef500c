#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest -q -x -p no:cacheprovider tests -m gpu 2>&1 | tail -3
for a in "112 10240 8192 0" "112 8192 8192 0 rms"; do timeout 120 python tools/epi_trace.py $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('N','K','acc_done','exit','epilogue_total','stores')})"; done
for Q in 5 7 9; do timeout 300 python tools/llama_verify_breakdown.py llama-2-70b $Q 190 16 2>&1 | grep -E "full"; done
