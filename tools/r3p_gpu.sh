#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest -q -p no:cacheprovider tests -m gpu > $O/r3p_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/r3p_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 python bench.py > $O/r3p_bench.json 2> $O/r3p_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/r3p_bench.json')); print(d['value'], d['e2e']['value'], d['mean_accepted_length'], d['verify_ms_mean'], d['draft_ms_mean'], d['roofline']['frac'], d['clocks'], d.get('warm_controllers',{}).get('value'), d['lossless_vs_greedy'], d['gpu_launches'])"
timeout 1200 python bench.py --impl reference > $O/r3p_bench_ref.json 2> $O/r3p_bench_ref.err; echo "ref rc=$?"; cat $O/r3p_bench_ref.json | head -c 400; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r3p_launches.csv python bench.py --steps 1 --warmup 0 > $O/r3p_ncu_bench.log 2>&1; echo "ncu rc=$?"
