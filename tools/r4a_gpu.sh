#!/bin/bash
# ncu --set full of the online-softmax tcgen05 attention (70B heads, B = 16,
# 4K cache, Q = 5) beside the row kernel, after the softmax rework
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"attention_(tc|rows)_kernel" -s 2 -c 2 \
  -o $O/r4a_attn4k python tools/ncu_attn.py 5 4096 > $O/r4a_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 $O/r4a_ncu.log
