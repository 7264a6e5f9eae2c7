#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -15 > gpurun_out/it2_tests.log
bash tools/variants.sh run 100 > gpurun_out/it2_variants.txt 2>&1
bash tools/variants.sh run 100 >> gpurun_out/it2_variants.txt 2>&1
cat gpurun_out/it2_tests.log gpurun_out/it2_variants.txt
