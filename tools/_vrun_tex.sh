#!/bin/bash
# A/B of environment knobs on the current library (two-stream / one-stream frame time).
for round in 1 2; do
for v in "NX_STREAM_PRIORITY=0" "NX_STREAM_PRIORITY=0 NX_PROBE_FRAMES=3" "NX_STREAM_PRIORITY=1 NX_PROBE_FRAMES=3" "NX_STREAM_PRIORITY=1 NX_PROBE_FRAMES=3 NX_TEXTURE_PATH=split2ts NX_TS_CTAS_PER_SM=3" "NX_STREAM_PRIORITY=0 NX_PROBE_FRAMES=3 NX_TEXTURE_PATH=split2ts NX_TS_CTAS_PER_SM=3" "NX_STREAM_PRIORITY=1 NX_PROBE_FRAMES=4 NX_TEXTURE_PATH=split2ts NX_TS_CTAS_PER_SM=3"; do
  echo "$v $(env $v timeout 300 python tools/stream_probe.py 2>/dev/null | head -2 | tr '\n' ' ')"
done; done
