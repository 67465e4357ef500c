#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py --no-cpu-baseline > $O/r2p_bench.json 2> $O/r2p_bench.err; echo "bench rc=$?"
MS_VERIFY_PRIORITY=1 timeout 900 python bench.py --no-cpu-baseline --fresh-steps 0 > $O/r2p_bench_vprio.json 2> $O/r2p_bench_vprio.err; echo "bench vprio rc=$?"
for f in r2p_bench r2p_bench_vprio; do python -c "
import json; d=json.load(open('$O/$f.json')); print('$f', d['value'], d['e2e']['value'], d['mean_accepted_length'], d['verify_ms_mean'], d['draft_ms_mean'], d['roofline']['frac'], d['clocks'])"; done
