"""Static LDL/STL count of the f32 W=32 CPB=2 step kernel grouped by source line range
(run tools/spills.sh first; it writes /tmp/spill.sass)."""
import re, sys
from collections import Counter
txt = open('/tmp/spill.sass').read()
fn = [p for p in re.split(r'//-+ \.text\.', txt) if p.startswith('_ZN3stp10k_env_stepIfLi32ELi2E')][0]
cur = None; c = Counter(); n = 0
for ln in fn.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    if re.search(r'/\*[0-9a-f]{4,}\*/', ln):
        n += 1
        if re.search(r'\b(STL|LDL)', ln):
            c[cur] += 1
print('instructions', n, 'spill instr', sum(c.values()))
for k, v in sorted(c.items(), key=lambda kv: -kv[1])[:int(sys.argv[1]) if len(sys.argv) > 1 else 20]:
    print(' ', v, k)
