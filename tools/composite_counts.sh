#!/bin/bash
# Rebuilds the composite / composite-backward kernels with pair counters and runs a
# forward + a training step.
set -e
make -s lib >/dev/null
for f in nx_composite nx_backward; do
/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 \
   --expt-relaxed-constexpr -DNX_COMPOSITE_COUNT -c -o build/obj/$f.o paper_2512_13796_b200/csrc/$f.cu
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2512_13796_b200/libnexel_b200.so \
   build/obj/*.o -Xlinker -Bsymbolic
python bench.py --steps 3 --warmup 3 --train-steps 1 --no-cpu-baseline 2>&1 | grep counts | tail -8
