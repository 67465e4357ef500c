#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest -q -p no:cacheprovider tests -m gpu > $O/r2ff_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/r2ff_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1200 python bench.py > $O/r2ff_bench.json 2> $O/r2ff_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/r2ff_bench.json')); print(d['value'], d['e2e']['value'], d['mean_accepted_length'], d['verify_ms_mean'], d['draft_ms_mean'], d['roofline']['frac'], d['clocks'], d['fresh_controllers']['value'], d['lossless_vs_greedy'])"
