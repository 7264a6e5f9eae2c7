#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_binning.py -q -x 2>&1 | tail -8 > gpurun_out/it3_tests.log
bash tools/variants.sh run 100 > gpurun_out/it3_variants.txt 2>&1
bash tools/variants.sh run 100 >> gpurun_out/it3_variants.txt 2>&1
cat gpurun_out/it3_tests.log gpurun_out/it3_variants.txt
