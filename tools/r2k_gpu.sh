#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
for B in 32 64; do
  timeout 1200 python bench.py --batch $B --no-cpu-baseline --fresh-steps 0 > $O/r2k_bench_b$B.json 2> $O/r2k_bench_b$B.err; echo "bench B=$B rc=$?"; tail -c 1200 $O/r2k_bench_b$B.json; tail -2 $O/r2k_bench_b$B.err
done
