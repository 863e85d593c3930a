O=gpurun_out/sel4
mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/gputests.log 2>&1; tail -2 $O/gputests.log
for w in c3 c5 c1; do python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
python bench.py --plan fixed16 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_fixed16.json 2> $O/bench_fixed16.err
python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
for f in $O/bench_*.json; do python -c "
import json
d=json.load(open('$f'))
print('$f', round(d['value'],1), round(d['ms_per_step']*1e3,1), {k:round(v*1e3,1) for k,v in d.get('kernels_ms',{}).items()})
"; done
