#!/bin/bash
# Per-kernel registers / spills of a .cu file (sm_100a).
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v -c "$1" -o /tmp/_regs.o 2>&1 | \
python3 -c "
import re,sys
cur=None
for line in sys.stdin:
    m=re.search(r\"entry function '([^']+)'\",line)
    if m: cur=m.group(1); continue
    m=re.search(r'(\d+) bytes spill stores',line)
    if m: spill=int(m.group(1)); continue
    m=re.search(r'Used (\d+) registers',line)
    if m and cur:
        k=re.search(r'kernelI(.*)EEv',cur)
        print(f'{m.group(1):>4} regs spill={spill:<4} {k.group(1) if k else cur}')
"
