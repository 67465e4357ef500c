#!/bin/bash
# diagnostic library with the attention_tc phase timers (-DATC_PROF)
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2402_15678_b200 import build as b; b.build()"
mkdir -p paper_2402_15678_b200/lib/ab build/prof
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 $EXTRA -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Iinclude -Ipaper_2402_15678_b200/csrc -DATC_PROF \
  -c paper_2402_15678_b200/csrc/attention_tc.cu -o build/prof/attention_tc${SUFFIX}.o
objs=$(ls build/obj/*.o | grep -v attention_tc.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2402_15678_b200/lib/ab/libminions_atcprof${SUFFIX}.so $objs build/prof/attention_tc${SUFFIX}.o
echo built
