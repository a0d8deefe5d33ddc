#!/bin/bash
# one summary line per bench log
for f in "$@"; do tail -n 1 $f | python -c "
import sys,json
try:
    d=json.loads(sys.stdin.readline())
except Exception as e:
    print('$f', 'no json'); sys.exit()
print('$f'.split('/')[-1], d['value'], d['ms_per_step'], 'step_roof', d['step_roofline']['frac'], 'attn', d['roofline']['frac'], {k:(v['avg_ms'],v['launches']) for k,v in d['kernels'].items()}, 'e2e', d['e2e'] and d['e2e']['value'])"; done
