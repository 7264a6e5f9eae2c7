#!/bin/bash
# Round-2 GPU session: fp64 peak, GPU suite, bench line, launch list, ncu of the
# binning stages and the composite (on the GPU box; outputs under gpurun_out/).
#   bash tools/gpu_round2.sh [tag] [skip_tests]
mkdir -p gpurun_out
TAG=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak_$TAG.json
if [ -z "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -rA 2>&1 | grep -v "^PASSED" | tail -60 > gpurun_out/gpu_tests_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --train-steps 0 > gpurun_out/ncu_bench_$TAG.log 2>&1
# binning stages of the 3rd frame + the composite, full sets (+ fp64 instruction counts)
FP64M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_fp64_pred_on.sum
timeout 600 ncu --set full --clock-control none --import-source on --metrics $FP64M \
  -k "regex:radix|scan_|emit|compact|rect_counts|preprocess" -s 160 -c 80 \
  -o gpurun_out/ncu_binning_$TAG -f python tools/prof_frame.py --frames 3 > gpurun_out/ncu_binning_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --metrics $FP64M \
  -k "regex:^composite_kernel" -s 2 -c 1 \
  -o gpurun_out/ncu_composite_$TAG -f python tools/prof_frame.py --frames 3 > gpurun_out/ncu_composite_$TAG.log 2>&1
tail -3 gpurun_out/gpu_tests_$TAG.log 2>/dev/null; cat gpurun_out/fp64_peak_$TAG.json; tail -c 600 gpurun_out/bench_$TAG.log
