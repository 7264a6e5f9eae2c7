#!/bin/bash
mkdir -p gpurun_out
VT=120 bash tools/variants.sh run 100 > gpurun_out/it7_variants.txt 2>&1
VT=120 bash tools/variants.sh run 100 >> gpurun_out/it7_variants.txt 2>&1
cat gpurun_out/it7_variants.txt
