#!/bin/bash
# Round-2 evidence on the GPU box: GPU suite, bench lines (config 2 with CPU baseline,
# config 4), reference arm, launch metrics of one frame, ncu of the composite kernels,
# the texture kernels and the binning kernels, CUPTI timelines.
mkdir -p gpurun_out
T=${1:-r02f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rA 2>&1 | grep -v "^PASSED" | tail -40 > gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.log 2>&1
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench4.log 2>&1
timeout 600 python tools/timeline.py --one-stream --out gpurun_out/${T}_tl1.json > gpurun_out/${T}_tl1.txt 2>&1
timeout 600 python tools/timeline.py --out gpurun_out/${T}_tl2.json > gpurun_out/${T}_tl2.txt 2>&1
bash tools/frame_metrics.sh ${T}
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:tex_|radix|emit|scan_|preprocess|redo" -s 40 -c 24 \
  -o gpurun_out/${T}_others -f python tools/prof_frame.py --frames 4 > gpurun_out/${T}_others.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --train-steps 0 > gpurun_out/${T}_ncu_bench.log 2>&1
tail -3 gpurun_out/${T}_tests.log; tail -c 400 gpurun_out/${T}_bench.log
# summaries on the box (the full `others` report alone is ~48 MB: gpurun returns <= 64 MiB)
python tools/ncu_table.py gpurun_out/${T}_others.ncu-rep > gpurun_out/${T}_others_table.txt 2>&1
python tools/ncu_summary.py gpurun_out/${T}_composite.ncu-rep > gpurun_out/${T}_composite_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/${T}_composite.ncu-rep 40 > gpurun_out/${T}_composite_lines.txt 2>&1
rm -f gpurun_out/${T}_others.ncu-rep gpurun_out/${T}_tl1.json gpurun_out/${T}_tl2.json
