#!/bin/bash
# Phase profile of nexel::render through the C++ drop-in at config 2 (F64 colour), with
# and without transparent huge pages for the FrameBuffers, and with glibc keeping freed
# pages (no mmap for large blocks).
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag; nproc
for v in "A=1" "NEXEL_DROPIN_NO_THP=1" "GLIBC_TUNABLES=glibc.malloc.mmap_max=0:glibc.malloc.trim_threshold=4000000000" "NEXEL_DROPIN_PRECISION=f32"; do
  echo "== $v"
  env $v NEXEL_DROPIN_PROFILE=1 timeout 300 build/dropin/bench_render 8 2>&1 | tail -3
done
