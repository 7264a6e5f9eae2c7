#!/bin/bash
mkdir -p gpurun_out
bash tools/variants.sh run 100 > gpurun_out/it5_variants.txt 2>&1
bash tools/variants.sh run 100 >> gpurun_out/it5_variants.txt 2>&1
cat gpurun_out/it5_variants.txt
