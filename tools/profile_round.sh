#!/usr/bin/env bash
# Profiling recipe (run on the GPU box via gpurun; one GPU, never multi-rank):
#   1. launch list of one bench step (cold-cache, serialised per-kernel times)
#   2. one `ncu --set full` capture of each of the two dominant kernels
# Outputs land in gpurun_out/; summaries are copied to profiles/ by hand.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > "$OUT/launches_bench.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:composite_kernel -s 1 -c 1 \
    -o "$OUT/prof_composite" python tools/prof_frame.py --frames 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:texture_tc_kernel -s 1 -c 1 \
    -o "$OUT/prof_texture" python tools/prof_frame.py --frames 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:preprocess_kernel -s 1 -c 1 \
    -o "$OUT/prof_preprocess" python tools/prof_frame.py --frames 2 > /dev/null 2>&1
echo done
