#!/bin/bash
mkdir -p gpurun_out
bash tools/variants.sh run 100 > gpurun_out/it1_variants.txt 2>&1
bash tools/variants.sh run 100 >> gpurun_out/it1_variants.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/it1_bench.log 2>&1
cat gpurun_out/it1_variants.txt; tail -c 600 gpurun_out/it1_bench.log
