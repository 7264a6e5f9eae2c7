#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py -q -x -k "textur or tensor or variant or config2" 2>&1 | tail -8 > gpurun_out/it4_tests.log
bash tools/variants.sh run 100 > gpurun_out/it4_variants.txt 2>&1
bash tools/variants.sh run 100 >> gpurun_out/it4_variants.txt 2>&1
cat gpurun_out/it4_tests.log gpurun_out/it4_variants.txt
