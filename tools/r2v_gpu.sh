#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1500 python bench.py --preset cfg5 --steps 2 --no-cpu-baseline --fresh-steps 0 > $O/r2v_bench_cfg5.json 2> $O/r2v_bench_cfg5.err; echo "cfg5 rc=$?"; tail -c 400 $O/r2v_bench_cfg5.json; tail -2 $O/r2v_bench_cfg5.err
timeout 900 python bench.py --target opt-13b --ssm opt-125m --schedule sequential --no-cpu-baseline --fresh-steps 0 > $O/r2v_bench_cfg2.json 2> $O/r2v_bench_cfg2.err; echo "cfg2 rc=$?"; tail -c 400 $O/r2v_bench_cfg2.json
timeout 900 python bench.py --preset cfg1 --no-cpu-baseline --fresh-steps 0 > $O/r2v_bench_cfg1.json 2> $O/r2v_bench_cfg1.err; echo "cfg1 rc=$?"; tail -c 400 $O/r2v_bench_cfg1.json
