#!/bin/bash
# Round-2 final evidence on one B200 (run through gpurun): GPU tests, bench
# lines of every workload, the reference arm, the launch list and ncu captures.
# One step = k_prepare, k_score_tma, k_select (+ fused worklist), k_attend_tma,
# k_merge_units; `--quick --steps 8 --warmup 3` runs 11 steps, so -s 55 -c 5
# captures the first untimed extra step, whose algorithmic attention bytes the
# quick line reports first in quick_attend_bytes_next_steps.
set -x
O=gpurun_out/r2f
mkdir -p $O
python -m pytest tests -m gpu -q -rA > $O/gputests.log 2>&1; tail -3 $O/gputests.log
python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
for w in c1 c3 c4 c5; do python bench.py --workload $w --steps 20 --warmup 5 > $O/bench_$w.json 2> $O/bench_$w.err; done
python bench.py --plan fixed16 --steps 50 --warmup 5 > $O/bench_fixed16.json 2> $O/bench_fixed16.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py --quick --steps 8 --warmup 3 > $O/quick.json 2> $O/quick.err
ncu --set full --import-source on --clock-control none -k regex:'k_attend|k_score|k_select|k_prepare|k_merge_units' -s 55 -c 5 \
    -o $O/step python bench.py --quick --steps 8 --warmup 3 > $O/step_quick.json 2> $O/step.err
ncu --set full --import-source on --clock-control none -k regex:'k_attend|k_score|k_select|k_prepare|k_merge_units' -s 55 -c 5 \
    -o $O/step_fixed16 python bench.py --quick --plan fixed16 --steps 8 --warmup 3 > $O/step_fixed16_quick.json 2> $O/step_fixed16.err
ncu --set full --clock-control none -k regex:k_meta_stream -c 1 -o $O/meta python bench.py --quick --steps 2 --warmup 3 > /dev/null 2> $O/meta.err
ncu --set full --import-source on --clock-control none -k regex:"k_feat|k_mlp" -s 6 -c 3 -o $O/pred python profiles/pred_profile.py 4 > /dev/null 2> $O/pred.err
python profiles/pred_timing.py > $O/pred_timing.json 2> $O/pred_timing.err
ls -la $O
# compute-sanitizer over the small end-to-end run (profiles/sanitizer/README.md)
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python profiles/sanitizer/small_step.py > $O/san_$t.log 2>&1
  tail -2 $O/san_$t.log
done
