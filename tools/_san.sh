#!/bin/bash
# compute-sanitizer over the config-1-sized render, full reports into gpurun_out/
mkdir -p gpurun_out
python - <<'PY' > /tmp/san.py
import re
src = open("tests/test_gpu_sanitizer.py").read()
print(re.search(r'_SCRIPT = r"""(.*?)"""', src, re.S).group(1))
PY
for tw in "memcheck forward" "racecheck forward" "memcheck backward"; do
  set -- $tw
  timeout 900 compute-sanitizer --tool $1 --print-limit 20 python /tmp/san.py $PWD $2 > gpurun_out/san_$1_$2.txt 2>&1
  echo "$1 $2 rc=$?"; grep -m3 -n "ERROR SUMMARY\|Invalid\|Race\|Error" gpurun_out/san_$1_$2.txt
done
