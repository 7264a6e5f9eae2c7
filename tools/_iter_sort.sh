#!/bin/bash
# binning parity + bench stage times after a sort change
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2; do
  timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --train-steps 0 > /tmp/b.log 2>&1
  python -c "
import json
for l in open('/tmp/b.log'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'stages', {k: round(v,3) for k,v in d['stages_ms'].items()})
"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sort_frame.csv python tools/prof_frame.py --frames 3 > /dev/null 2>&1
python tools/frame_dram.py gpurun_out/sort_frame.csv 2>&1 | head -20
