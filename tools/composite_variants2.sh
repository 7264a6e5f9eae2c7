# Rebuilds the composite kernel with (min CTAs/SM, B1 unroll) variants and benches each.
set -e
for v in "10 1" "8 2" "8 1" "7 2"; do
  set -- $v
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 \
     --expt-relaxed-constexpr -DNX_COMPOSITE_MINB=$1 -DNX_COMPOSITE_B1_UNROLL=$2 \
     -c -o build/obj/nx_composite.o paper_2512_13796_b200/csrc/nx_composite.cu
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2512_13796_b200/libnexel_b200.so \
     build/obj/*.o -Xlinker -Bsymbolic
  echo "== minb $1 unroll $2"
  python bench.py --steps 150 --no-cpu-baseline --train-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['stages_ms']['composite'],3))"
done
