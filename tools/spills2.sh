#!/bin/bash
# spill sites of a kernel (regex on mangled name) in the f32 build
PAT=${1:-k_solveIfLi32ELi2E}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -cubin $STP_NVCC_EXTRA -I/root/repo/include -I/root/repo/paper_1810_05762_b200/csrc /root/repo/paper_1810_05762_b200/csrc/sim_step_f32.cu -o /tmp/spill.cubin 2>/dev/null
nvdisasm -g /tmp/spill.cubin 2>/dev/null > /tmp/spill.sass
PAT=$PAT python3 - <<'PY'
import re, os
from collections import Counter
txt=open('/tmp/spill.sass').read()
pat=os.environ['PAT']
for p in re.split(r'//-+ \.text\.', txt):
    if pat not in p[:80]: continue
    cur=None; c=Counter(); tot=0; n=0; ld=Counter()
    for ln in p.splitlines():
        m=re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m: cur=(m.group(1).split('/')[-1], int(m.group(2))); continue
        if re.search(r'/\*[0-9a-f]{4,}\*/', ln): n+=1
        if re.search(r'\b(STL|LDL)', ln): c[cur]+=1; tot+=1
        if re.search(r'\bLDG', ln): ld[cur]+=1
    print(p[:60], 'instructions', n, 'spill instr', tot)
    for k,v in sorted(c.items(), key=lambda kv:-kv[1])[:14]: print('  spill',v,k)
    break
PY
