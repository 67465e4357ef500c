#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 300 python tools/draft_step.py 200 16 3 > $O/r2i_draft_step.jsonl 2>&1; echo "draft rc=$?"; cat $O/r2i_draft_step.jsonl | tail -4
timeout 1200 python tools/partition_ab.py "draft_pdl=1;draft_pdl=0" 6 2 > $O/r2i_pdl_ab.jsonl 2> $O/r2i_pdl_ab.err; echo "ab rc=$?"; cat $O/r2i_pdl_ab.jsonl; tail -3 $O/r2i_pdl_ab.err
