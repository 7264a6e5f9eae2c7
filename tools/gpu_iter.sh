#!/bin/bash
# One build -> measure iteration on the GPU box (outputs under gpurun_out/<tag>_*):
#   bash tools/gpu_iter.sh TAG "pytest selection (or -)" [ncu kernel regex (or -)] [extra command]
mkdir -p gpurun_out
TAG=$1; SEL=$2; KRE=${3:--}; EXTRA=${4:-}
if [ "$SEL" != "-" ]; then
  timeout 1500 python -m pytest $SEL -x -q -rA 2>&1 | grep -v "^PASSED" | tail -40 > gpurun_out/${TAG}_tests.log
  tail -3 gpurun_out/${TAG}_tests.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --train-steps 0 > gpurun_out/${TAG}_bench.log 2>&1
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
for l in open(f"gpurun_out/{tag}_bench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "stages", {k: round(v, 3) for k, v in d["stages_ms"].items()})
PY
if [ "$KRE" != "-" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on \
    -k "regex:$KRE" -s 2 -c 1 -o gpurun_out/${TAG}_ncu -f python tools/prof_frame.py --frames 3 > gpurun_out/${TAG}_ncu.log 2>&1
  python tools/ncu_summary.py gpurun_out/${TAG}_ncu.ncu-rep | head -24
fi
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
