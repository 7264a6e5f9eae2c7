#!/bin/bash
# ncu --set full captures of the backward kernels (config 2, one launch each).
mkdir -p gpurun_out
TAG=${1:-cur}
for K in ${KERNELS:-composite_bwd_kernel scatter_table_kernel mlp_bwd_tc_kernel}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^$K" -s 1 -c 1 \
     -o gpurun_out/ncu_${K}_${TAG} -f python tools/bwd_timing.py > gpurun_out/ncu_${K}_${TAG}.log 2>&1
  tail -1 gpurun_out/ncu_${K}_${TAG}.log
done
