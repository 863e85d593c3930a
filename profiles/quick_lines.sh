#!/bin/bash
# Quick bench lines of every workload without the CPU baseline (iteration aid).
O=gpurun_out/ql
mkdir -p $O
python bench.py --no-cpu-baseline > $O/c2.json 2> $O/c2.err
for w in c1 c3 c4 c5; do python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > $O/$w.json 2> $O/$w.err; done
python bench.py --plan fixed16 --steps 50 --warmup 5 --no-cpu-baseline > $O/fixed16.json 2> $O/fixed16.err
for w in c2 c1 c3 c4 c5 fixed16; do python -c "
import json
d=[json.loads(l) for l in open('$O/$w.json') if l.startswith('{')][-1]
print('$w', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],3), {k: round(v*1e3,1) for k,v in d.get('kernels_ms',{}).items()}, 'pred', (d.get('predictor_path') or {}).get('value'))
"; done
