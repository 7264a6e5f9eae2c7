#!/bin/bash
# Build (here) or measure (on the GPU box) compile-time variants of one kernel file.
#   bash tools/variants.sh build SRC "name1:-DX=1 -DY=2" "name2:..."   -> build/variants/<name>.so
#   bash tools/variants.sh run [steps]                                  -> bench each variant
set -e
mode=$1; shift
NV="/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr"
if [ "$mode" = build ]; then
  src=$1; shift
  base=$(basename $src .cu)
  mkdir -p build/variants
  for v in "$@"; do
    name=${v%%:*}; defs=${v#*:}
    mkdir -p build/variants/obj_$name
    $NV $defs -c -o build/variants/obj_$name/$base.o $src
    objs=$(ls build/obj/*.o | grep -v "/$base.o$")
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/$name.so \
      $objs build/variants/obj_$name/$base.o -Xlinker -Bsymbolic
    echo "built $name ($defs)"
  done
else
  steps=${1:-60}
  cp paper_2512_13796_b200/libnexel_b200.so /tmp/main.so
  for so in build/variants/*.so; do
    cp $so paper_2512_13796_b200/libnexel_b200.so
    echo "== $(basename $so .so): $(timeout 300 python bench.py --steps $steps --warmup 5 --no-cpu-baseline --train-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), {k: round(v,3) for k,v in d['stages_ms'].items()})")"
  done
  cp /tmp/main.so paper_2512_13796_b200/libnexel_b200.so
fi
