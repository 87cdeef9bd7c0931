#!/bin/bash
# ptxas register / spill summary for the evaluation kernels (dev tool)
cd "$(dirname "$0")/.." && /usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include \
  -gencode arch=compute_100a,code=sm_100a -fmad=false -Xptxas -v -c paper_2011_11880_b200/csrc/pf_eval.cu \
  -o /tmp/_regs.o 2>&1 | python3 -c "
import re,sys
lines=sys.stdin.read().splitlines()
name=None
for i,l in enumerate(lines):
    m=re.search(r'Function properties for (\S+)',l)
    if m: name=m.group(1); spill=lines[i+1].strip(); continue
    m=re.search(r'Used (\d+) registers',l)
    if m and name and ('k_eval' in name):
        short=re.sub(r'_ZN2pf\w+?_pf_eval_cu_\w+?(\d+k_eval)', r'\1', name)[:60]
        print(f'{short:60s} regs={m.group(1):>4}  {spill}')
        name=None
"
