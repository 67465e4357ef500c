#!/bin/bash
# final check of the round's last code: GPU suite, smoke, bench line
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/r4d_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/r4d_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/r4d_smoke.log 2>&1; tail -1 $O/r4d_smoke.log
python bench.py > $O/r4d_bench.json 2> $O/r4d_bench.err; echo "bench rc=$?"
python bench.py --impl reference > $O/r4d_bench_reference.json 2> $O/r4d_bench_reference.err; echo "ref rc=$?"
