#!/bin/bash
# One GPU call that regenerates the round's measurement evidence under gpurun_out/prof/:
# bench line (c1, CPU baseline, e2e), launch list, per-config event timelines, ncu --set full of
# the dominant kernels. Summarised into profiles/ by hand (see profiles/README.md).
cd "$(dirname "$0")/.."
O=gpurun_out/prof
mkdir -p $O
timeout 400 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
for c in c2 c3 c4; do timeout 300 python bench.py --config $c --steps 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in c1 c2 c3 c4; do timeout 200 python tools/profile_step.py --config $c --reps 3 > $O/events_$c.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches_c1.csv 2> $O/launches_c1.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:far_group -s 20 -c 1 -o $O/far_c1_mid python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tile_diag_lines -s 22 -c 1 -o $O/lines_c1_mid python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:far_group -s 28 -c 1 -o $O/far_c3_mid python tools/profile_step.py --config c3 --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:zgemm_dmma -s 2 -c 1 -o $O/zgemm_c1 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
echo done > $O/done
