#!/bin/bash
# texture parity + bench stage times + per-kernel launch times after a gather change
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "textur or config2 or smoke or precision or backward or field" 2>&1 | tail -3
for rep in 1 2; do
  timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --train-steps 0 > /tmp/b.log 2>&1
  python -c "
import json
for l in open('/tmp/b.log'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'stages', {k: round(v,3) for k,v in d['stages_ms'].items()})
"
done
timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts.sum --clock-control none -k regex:tex_features_img -s 2 -c 1 python tools/prof_frame.py --frames 3 2>&1 | grep -E "duration|wavefronts|sectors" | head
