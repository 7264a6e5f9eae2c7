#!/bin/bash
# A/B of texture-pass variants (NX_TEXTURE_PATH / NX_TS_CTAS_PER_SM) on the current library.
for round in 1 2; do
for v in "NX_TEXTURE_PATH=split2" "NX_TEXTURE_PATH=split2ts NX_TS_CTAS_PER_SM=1" "NX_TEXTURE_PATH=split2ts NX_TS_CTAS_PER_SM=2" "NX_TEXTURE_PATH=split2ts NX_TS_CTAS_PER_SM=3"; do
  echo "$v $(env $v timeout 300 python tools/stream_probe.py 2>/dev/null | head -2 | tr '\n' ' ')"
done; done
