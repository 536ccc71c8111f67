#!/bin/bash
# where do spills (STL/LDL) of the f32 W=32 CPB=2 kernel come from?
# same per-source flags as build.py PER_SOURCE for the fp32 TU
STP_NVCC_EXTRA=${STP_NVCC_EXTRA:--ftz=true -prec-div=false -prec-sqrt=false}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -cubin $STP_NVCC_EXTRA -I/root/repo/include -I/root/repo/paper_1810_05762_b200/csrc /root/repo/paper_1810_05762_b200/csrc/sim_step_f32.cu -o /tmp/spill.cubin 2>/dev/null
nvdisasm -g /tmp/spill.cubin 2>/dev/null > /tmp/spill.sass
python3 - <<'PY'
import re
from collections import Counter
txt=open('/tmp/spill.sass').read()
for p in re.split(r'//-+ \.text\.', txt):
    if not p.startswith('_ZN3stp10k_env_stepIfLi32ELi2E'): continue
    cur=None; c=Counter(); tot=0; n=0
    for ln in p.splitlines():
        m=re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m: cur=(m.group(1).split('/')[-1], int(m.group(2))); continue
        if re.search(r'/\*[0-9a-f]{4,}\*/', ln): n+=1
        if re.search(r'\b(STL|LDL)', ln): c[cur]+=1; tot+=1
    print('instructions', n, 'spill instr', tot)
    for k,v in sorted(c.items(), key=lambda kv:-kv[1])[:12]: print(' ',v,k)
PY
