#!/bin/bash
# round-2 closing run: GPU suite, smoke, bench line, bf16 numerics report,
# ncu launch list of prefill + 3 decode rounds (kernel shares of a round)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/r4b_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/r4b_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/r4b_smoke.log 2>&1; tail -1 $O/r4b_smoke.log
python bench.py > $O/r4b_bench.json 2> $O/r4b_bench.err; echo "bench rc=$?"
timeout 900 python tools/bf16_numerics.py --big --out $O/r4b_bf16_numerics.jsonl > $O/r4b_numerics.log 2>&1; echo "numerics rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r4b_launches.csv \
  python tools/profile_round.py 3 > $O/r4b_ncu_round.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py $O/r4b_launches.csv --after wide_kernel > $O/r4b_launch_summary.txt 2>&1; head -25 $O/r4b_launch_summary.txt
