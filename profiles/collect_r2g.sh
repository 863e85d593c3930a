#!/bin/bash
# Round-2 closing evidence of the final code on one B200 (through gpurun):
# GPU tests, smoke, and the full bench line (e2e, roofline, cpu_baseline,
# in-run parity) of every workload.
O=gpurun_out/r2g
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python -m pytest tests -m gpu -q -rA > $O/gputests.log 2>&1; tail -1 $O/gputests.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
for w in c1 c3 c4 c5; do python bench.py --workload $w --steps 20 --warmup 5 > $O/bench_$w.json 2> $O/bench_$w.err; done
python bench.py --plan fixed16 --steps 50 --warmup 5 > $O/bench_fixed16.json 2> $O/bench_fixed16.err
for f in $O/bench_*.json; do python -c "
import json
d=json.load(open('$f'))
p=d.get('parity') or {}
print('$f', round(d['value'],1), round((d.get('e2e') or {}).get('value',0),1), round((d.get('roofline') or {}).get('frac',0),3), p.get('selection_mismatches'), p.get('max_rel_err'), (d.get('clocks') or {}).get('reasons'))
"; done
