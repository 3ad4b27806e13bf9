#!/bin/bash
# One GPU call that regenerates the round's measurement evidence under gpurun_out/prof/: bench
# lines (c1 with the CPU baseline and e2e; c2-c4), the sharded engine at one rank (c3, c4), the
# reference arm on full c1 (2 steps), per-config event timelines, the c1 launch list, and ncu
# --set full captures of the dominant kernels. Summarised into profiles/ (profiles/README.md).
cd "$(dirname "$0")/.."
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
for c in c2 c3 c4; do timeout 400 python bench.py --config $c --steps 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in c3 c4; do timeout 400 python bench.py --sharded --config $c --steps 3 --warmup 2 > $O/bench_sharded1_$c.json 2> $O/bench_sharded1_$c.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/reference_c1.json 2> $O/reference_c1.err
for c in c1 c2 c3 c4; do timeout 300 python tools/profile_step.py --config $c --reps 3 > $O/events_$c.txt 2>&1; done
NDS_SOLVE_TRACE=1 timeout 300 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2> $O/trace_c1.txt
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-verify > $O/launches_c1.csv 2> $O/launches_c1.err
timeout 400 ncu --set full --clock-control none --import-source on -k regex:zgemm_tma -s 1 -c 1 -o $O/zgemm_tma_c1 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:zgemm_dmma -s 0 -c 1 -o $O/zgemm_dmma_c1 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:far_group -s 20 -c 1 -o $O/far_c1_mid python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:tile_diag_lines -s 22 -c 1 -o $O/lines_c1_mid python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:binary_pass -s 1 -c 1 -o $O/binary_pass_c4 python tools/profile_step.py --config c4 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:binary_tile_solve -s 8 -c 1 -o $O/binary_solve_c4 python tools/profile_step.py --config c4 --reps 1 > /dev/null 2>&1
echo done > $O/done
