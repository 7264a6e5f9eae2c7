#!/bin/bash
# One `ncu --set full` capture per hot kernel (config 2, a warm view), for profiles/.
# Usage (on the GPU box): bash tools/profile_round.sh [tag]
mkdir -p gpurun_out
TAG=${1:-cur}
for K in composite_kernel tex_features_kernel tex_mlp_kernel preprocess_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:^$K" -s 3 -c 1 \
     -o gpurun_out/ncu_${K}_${TAG} -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --train-steps 0 \
     > gpurun_out/ncu_${K}_${TAG}.log 2>&1
  tail -1 gpurun_out/ncu_${K}_${TAG}.log
done
