#!/bin/bash
# final lines after the prefill-attention changes: smoke, headline bench, cfg5, cfg2
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/r4k_smoke.log 2>&1; tail -1 $O/r4k_smoke.log
python bench.py > $O/r4k_bench.json 2> $O/r4k_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --preset cfg5 --steps 2 --warmup 3 > $O/r4k_cfg5.json 2> $O/r4k_cfg5.err; echo "cfg5 rc=$?"
timeout 600 python bench.py --preset cfg2 > $O/r4k_cfg2.json 2> $O/r4k_cfg2.err; echo "cfg2 rc=$?"
