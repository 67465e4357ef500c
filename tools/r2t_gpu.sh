#!/bin/bash
# round-2 evidence batch: bench line, ncu of the small kernels / drafter step / verify layer
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1200 python bench.py > $O/r2t_bench.json 2> $O/r2t_bench.err; echo "bench rc=$?"; tail -c 600 $O/r2t_bench.json
# vote / greedy accept (argmax over the logits + commit), full sets
timeout 600 ncu --set full --clock-control none -k regex:"vote|accept|argmax" -c 40 -o /tmp/va python tools/ncu_small.py va > /dev/null 2>&1; echo "ncu va rc=$?"
ncu -i /tmp/va.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed > $O/r2t_ncu_vote_accept.csv 2>/dev/null
# drafter decode step, co-resident shapes: every kernel of the third step
timeout 900 ncu --set full --clock-control none -s 130 -c 70 -o /tmp/dr python tools/ncu_small.py draftco > /dev/null 2>&1; echo "ncu draft rc=$?"
ncu -i /tmp/dr.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active > $O/r2t_ncu_draft_step.csv 2>/dev/null
# one 70B verify layer (Q = 7): the four GEMMs + GQA attention
timeout 900 ncu --set full --clock-control none -k regex:"linear_kernel|attention_rows" -s 800 -c 6 -o /tmp/vl python tools/verify_one.py 7 190 > /dev/null 2>&1; echo "ncu verify rc=$?"
ncu -i /tmp/vl.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,launch__registers_per_thread > $O/r2t_ncu_verify_layer.csv 2>/dev/null
ncu -i /tmp/vl.ncu-rep --page details --csv > $O/r2t_ncu_verify_layer_details.csv 2>/dev/null
ls -la $O/r2t_*
