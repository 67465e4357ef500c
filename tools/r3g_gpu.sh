#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest -q -p no:cacheprovider tests -m gpu > $O/r3g_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r3g_pytest.log
timeout 1200 python tools/partition_ab.py "tc_attention=0;tc_attention=2" 6 2 2>&1 | grep rep | tee $O/r3g_tc_ab.jsonl
timeout 1200 python bench.py > $O/r3g_bench.json 2> $O/r3g_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/r3g_bench.json')); print(d['value'], d['e2e']['value'], d['mean_accepted_length'], d['verify_ms_mean'], d['draft_ms_mean'], d['roofline']['frac'], d['clocks'], d.get('warm_controllers',{}).get('value'), d['lossless_vs_greedy'])"
