#!/bin/bash
# ncu full captures of the two verify attention kernels at Q=7 ctx 190
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"attention_(tc|rows)_kernel" -s 2 -c 2 \
  -o $O/r3a_attn python tools/ncu_attn.py 7 190 > $O/r3a_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 $O/r3a_ncu.log
timeout 300 python tools/attn_tc_ab.py > $O/r3a_attn_tc_ab.jsonl 2>&1; cat $O/r3a_attn_tc_ab.jsonl
