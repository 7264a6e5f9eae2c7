#!/bin/bash
# ptxas register / spill summary of one .cu file's kernels: [REGS_FLAGS=-D...] bash tools/regs.sh FILE [name regex]
/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 \
  --expt-relaxed-constexpr $REGS_FLAGS -Xptxas -v -c -o /tmp/regs_$$.o "$1" 2>&1 | python3 -c "
import re, sys, subprocess
pat = re.compile(sys.argv[1])
name = None
for l in sys.stdin:
    m = re.search(r\"Compiling entry function '(\w+)'\", l)
    if m:
        name = subprocess.run(['c++filt', m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r'nx::\(anonymous namespace\)::', '', name)
    m = re.search(r'(\d+) bytes spill stores, (\d+) bytes spill loads', l)
    if m and name: spill = m.groups()
    m = re.search(r'Used (\d+) registers', l)
    if m and name and pat.search(name):
        print(f'{m.group(1):>4} regs  spill {spill[0]:>4}/{spill[1]:<4} {name[:110]}')
" "${2:-.}"
rm -f /tmp/regs_$$.o
