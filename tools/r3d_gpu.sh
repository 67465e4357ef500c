#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
for lib in atcprof atcprof_fx; do for c in "7 190" "13 190"; do
echo -n "$lib "; MS_LIB=paper_2402_15678_b200/lib/ab/libminions_$lib.so timeout 300 python tools/atc_prof.py $c 2>&1 | tail -1
done; done | tee $O/r3e_atc_prof.jsonl
