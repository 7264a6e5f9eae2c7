#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_download.py -q -x -s 2>&1 | tail -6 > gpurun_out/it6_tests.log
bash tools/variants.sh run 100 > gpurun_out/it6_variants.txt 2>&1
bash tools/variants.sh run 100 >> gpurun_out/it6_variants.txt 2>&1
cat gpurun_out/it6_tests.log gpurun_out/it6_variants.txt
