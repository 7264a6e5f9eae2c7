#!/bin/bash
# Launch list (ncu gpu__time_duration) of bench.py with 4 timed training steps; the
# summary divides by 4 (forward frames of the frame benchmark are included too).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/train_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --train-steps 4 > gpurun_out/train_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/train_launches.csv 4 | head -${1:-40}
