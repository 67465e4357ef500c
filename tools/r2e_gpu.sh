#!/bin/bash
# round-2 GPU batch (re-entry): full GPU tests, bench both arms, launch list of the bench
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/r2e_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2e_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/r2e_pytest_gpu.log
timeout 900 python bench.py > $O/r2e_bench.json 2> $O/r2e_bench.err; echo "bench rc=$?"; tail -c 3000 $O/r2e_bench.json; tail -3 $O/r2e_bench.err
timeout 900 python bench.py --impl reference > $O/r2e_bench_ref.json 2> $O/r2e_bench_ref.err; echo "ref rc=$?"; tail -c 1500 $O/r2e_bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file $O/r2e_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc=$?"
gzip -f $O/r2e_launches.csv
du -sh $O
