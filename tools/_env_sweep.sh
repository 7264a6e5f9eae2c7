#!/bin/bash
# runtime-knob sweep of the final build (200 frames each, two passes)
for rep in 1 2; do
for v in "NX_NONE=1" "NX_STREAM_PRIORITY=0" "NX_TS_CTAS_PER_SM=3" "NX_TEXTURE_PATH=split2"; do
  env $v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --train-steps 0 > /tmp/b.log 2>&1
  echo "$v $(python -c "
import json
for l in open('/tmp/b.log'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],1), 'e2e', round(d['e2e']['value'],1))
")"
done; done
