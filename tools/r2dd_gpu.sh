#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1200 python bench.py > $O/r2dd_bench.json 2> $O/r2dd_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/r2dd_bench.json')); print(d['value'], d['e2e']['value'], d['mean_accepted_length'], d['verify_ms_mean'], d['draft_ms_mean'], d['roofline']['frac'], d['clocks'], d['fresh_controllers']['value'])"
