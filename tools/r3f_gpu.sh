#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_attention_tc_gpu.py > $O/r3f_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/r3f_pytest.log
for c in "7 190" "13 190"; do
MS_LIB=paper_2402_15678_b200/lib/ab/libminions_atcprof.so timeout 300 python tools/atc_prof.py $c 2>&1 | tail -1
done | tee $O/r3f_atc_prof.jsonl
timeout 300 python tools/attn_tc_ab.py "5:190,7:190,9:190,13:190,7:300" > $O/r3f_attn_tc_ab.jsonl 2>&1; cat $O/r3f_attn_tc_ab.jsonl
