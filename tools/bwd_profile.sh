#!/bin/bash
# Launch list (ncu gpu__time_duration) of 2 forward+backward steps at config 2.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bwd_launches.csv \
    python tools/bwd_timing.py > gpurun_out/bwd_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/bwd_launches.csv 14 | head -30
