O=gpurun_out/sel
mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/gputests.log 2>&1; tail -3 $O/gputests.log
for w in c1 c3 c5; do python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
for f in $O/bench_*.json; do python -c "
import json,sys
d=json.load(open('$f'))
print('$f', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k:round(v*1e3,1) for k,v in d.get('kernels_ms',{}).items()}, d.get('parity'), (d.get('graph_replay') or {}).get('value'))
"; done
