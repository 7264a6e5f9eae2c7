#!/bin/bash
# Rebuilds the composite kernel with (chunk, sub, min CTAs/SM) variants and benches each.
set -e
for v in "128 8 8" "128 4 10" "64 4 12" "64 2 16" "128 4 8"; do
  set -- $v
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 \
     --expt-relaxed-constexpr -DNX_COMPOSITE_CHUNK=$1 -DNX_COMPOSITE_SUB=$2 -DNX_COMPOSITE_MINB=$3 \
     -c -o build/obj/nx_composite.o paper_2512_13796_b200/csrc/nx_composite.cu
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2512_13796_b200/libnexel_b200.so \
     build/obj/*.o -Xlinker -Bsymbolic
  echo "== chunk $1 sub $2 minb $3"
  python bench.py --steps 100 --no-cpu-baseline --train-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['stages_ms'])"
done
