#!/bin/bash
# Registers / spills of the fused kernels: scripts/regs.sh [extra nvcc flags]
cd "$(dirname "$0")/../paper_2204_01722_b200/csrc"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include -I. \
  --expt-relaxed-constexpr -Xptxas -v "$@" -c fused_apply.cu -o /tmp/fa_regs.o 2>&1 | python3 -c "
import sys,re
cur=None; sp='?'
for l in sys.stdin:
    m=re.search(r\"Compiling entry function '(\S+)'\",l)
    if m: cur=re.sub(r'.*?(fused_\w+kernel)ILi(\d)ELi(\d).*',r'\1<\2,\3>',m.group(1)); continue
    m=re.search(r'(\d+) bytes spill stores',l)
    if m and cur: sp=m.group(1)
    m=re.search(r'Used (\d+) registers',l)
    if m and cur: print(cur.split('3')[-1] if False else cur[-30:], 'regs',m.group(1),'spill',sp); cur=None
    if 'error' in l: print(l.strip())
"
