#!/bin/bash
# ncu --set full of one 70B verify layer (Q = 7, M = 112) on the round's final code
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum"
timeout 1200 ncu --set full --clock-control none -k regex:"linear_kernel|linear_gated_kernel|attention_tc_short" -s 807 -c 5 -o /tmp/vl python tools/verify_layer_ncu.py 7 > $O/r4e_ncu_verify.log 2>&1; echo "ncu verify rc=$?"
ncu -i /tmp/vl.ncu-rep --page raw --csv --metrics $M > $O/r4e_ncu_verify_layer.csv 2>/dev/null
tail -2 $O/r4e_ncu_verify.log
