#!/bin/bash
# Per-kernel DRAM bytes, duration and fp64 instruction counts of one config-2 frame
# (the 3rd rendered by tools/prof_frame.py), plus a full-set capture of the composite.
#   bash tools/frame_metrics.sh TAG   -> gpurun_out/TAG_frame.csv, TAG_composite.ncu-rep
mkdir -p gpurun_out
TAG=${1:-r02}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${TAG}_frame.csv \
  python tools/prof_frame.py --frames 3 > gpurun_out/${TAG}_frame.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --metrics $M -k "regex:^composite_kernel" -s 2 -c 1 \
  -o gpurun_out/${TAG}_composite -f python tools/prof_frame.py --frames 3 > gpurun_out/${TAG}_composite.log 2>&1
