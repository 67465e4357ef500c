#!/bin/bash
# tcgen05 prefill attention (query tiles): GPU suite, headline bench, cfg5
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/r4g_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/r4g_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/r4g_smoke.log 2>&1; tail -1 $O/r4g_smoke.log
python bench.py > $O/r4g_bench.json 2> $O/r4g_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --preset cfg5 --steps 2 --warmup 3 > $O/r4g_cfg5.json 2> $O/r4g_cfg5.err; echo "cfg5 rc=$?"
python tools/prefill_attn_ab.py > $O/r4g_prefill_attn_ab.jsonl 2>&1
