#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"attention_(tc_short|rows)_kernel" -s 2 -c 2 \
  -o $O/r3i_attn python tools/ncu_attn.py 7 190 > $O/r3i_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 $O/r3i_ncu.log
