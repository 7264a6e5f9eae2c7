#!/bin/bash
# e2e vs the number of streaming-copy CTAs (nx_frame_download)
for rep in 1 2; do
for v in 4 8 16 2; do
  NX_COPY_CTAS=$v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --train-steps 0 > /tmp/b.log 2>&1
  echo "copy_ctas=$v $(python -c "
import json
for l in open('/tmp/b.log'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['e2e'].get('roofline',{}).get('frac'))
")"
done; done
