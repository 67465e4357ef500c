#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum"
timeout 900 ncu --set full --clock-control none -k regex:"gemv|attention_decode|argmax|embed|linear_kernel" -s 126 -c 63 -o /tmp/dr python tools/ncu_small.py draftco > $O/r2u_ncu_draft.log 2>&1; echo "ncu draft rc=$?"
ncu -i /tmp/dr.ncu-rep --page raw --csv --metrics $M > $O/r2u_ncu_draft_step.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:"linear_kernel|attention_rows" -s 401 -c 6 -o /tmp/vl python tools/verify_one.py 7 190 > $O/r2u_ncu_verify.log 2>&1; echo "ncu verify rc=$?"
ncu -i /tmp/vl.ncu-rep --page raw --csv --metrics $M > $O/r2u_ncu_verify_layer.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:"linear_kernel" -s 1 -c 1 -o /tmp/g320 python tools/gemm_one.py 320 57344 8192 2 > /dev/null 2>&1; echo "ncu gu320 rc=$?"
ncu -i /tmp/g320.ncu-rep --page raw --csv --metrics $M > $O/r2u_ncu_gateup_m320.csv 2>/dev/null
ls -la $O/r2u_*
