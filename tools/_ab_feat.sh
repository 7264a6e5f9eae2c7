#!/bin/bash
# A/B of the feature-gather slot mapping (tile-major default vs NX_FEAT_MAP=row) + texture parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "textur or config2 or smoke or precision" 2>&1 | tail -3
for rep in 1 2; do
for v in "NX_FEAT_MAP=tile" "NX_FEAT_MAP=row"; do
  env $v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --train-steps 0 > /tmp/b.log 2>&1
  echo "$v $(python -c "
import json
for l in open('/tmp/b.log'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'stages', {k: round(v,3) for k,v in d['stages_ms'].items()})
")"
done; done
timeout 300 ncu --set full --clock-control none -k regex:tex_features_img -s 3 -c 1 -o gpurun_out/feat_tile -f python tools/prof_frame.py --frames 3 > /dev/null 2>&1
NX_FEAT_MAP=row timeout 300 ncu --set full --clock-control none -k regex:tex_features_img -s 3 -c 1 -o gpurun_out/feat_row -f python tools/prof_frame.py --frames 3 > /dev/null 2>&1
python tools/ncu_table.py gpurun_out/feat_tile.ncu-rep gpurun_out/feat_row.ncu-rep 2>&1 | tail -5
