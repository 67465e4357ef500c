#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests -m gpu > $O/r2q_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/r2q_pytest.log
timeout 300 python tools/draft_step.py 200 16 3 2>&1 | head -1
timeout 900 python bench.py --no-cpu-baseline --fresh-steps 0 > $O/r2q_bench.json 2> $O/r2q_bench.err; echo "bench rc=$?"
MS_VERIFY_PRIORITY=1 timeout 900 python bench.py --no-cpu-baseline --fresh-steps 0 > $O/r2q_bench_vprio.json 2> $O/r2q_bench_vprio.err; echo "bench vprio rc=$?"
for f in r2q_bench r2q_bench_vprio; do python -c "
import json; d=json.load(open('$O/$f.json')); print('$f', d['value'], d['e2e']['value'], d['mean_accepted_length'], d['verify_ms_mean'], d['draft_ms_mean'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['lossless_vs_greedy'])"; done
