#!/bin/bash
# C1 evidence (f32 warp-stream attention): bench line, launch list, ncu captures.
set -x
O=gpurun_out/c1f
mkdir -p $O
# (bench line: profiles/collect_r2f.sh or python bench.py --workload c1)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_c1.csv python bench.py --workload c1 --quick --steps 8 --warmup 3 > $O/quick_c1.json 2> $O/quick_c1.err
ncu --set full --import-source on --clock-control none -k regex:'k_attend_f32w|k_merge_chunks|k_approx|k_select|k_prepare' -s 55 -c 5 \
    -o $O/step_c1 python bench.py --workload c1 --quick --steps 8 --warmup 3 > $O/step_c1_quick.json 2> $O/step_c1.err
ls -la $O
