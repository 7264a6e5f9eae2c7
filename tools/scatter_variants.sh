# Rebuilds the field backward with scatter_table_kernel min-CTAs/SM variants (register
# caps) and times the training step for each.
set -e
for m in 1 10 12 16; do
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 \
     --expt-relaxed-constexpr -DNX_SCATTER_MINB=$m -Xptxas -v \
     -c -o build/obj/nx_field_backward_tc.o paper_2512_13796_b200/csrc/nx_field_backward_tc.cu 2>&1 | grep -A1 "scatter_table" | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' '
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2512_13796_b200/libnexel_b200.so \
     build/obj/*.o -Xlinker -Bsymbolic
  echo "== minb $m"
  for i in 1 2; do
    python bench.py --steps 10 --warmup 5 --no-cpu-baseline --train-steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); t=d['train_step']; print(round(t['ms_per_step'],3), round(t['losses_and_backward_ms'],3))"
  done
done
