#!/bin/bash
# One GPU call that regenerates the round's measurement evidence under gpurun_out/prof/: bench
# lines (c1 with the CPU baseline and e2e; c2-c4), the sharded engine at one rank (c3, c4), the
# reference arm on full c1 (2 steps), per-config event timelines, the c1 launch list, plan-creation
# times, and ncu --set full captures of the dominant kernels. Summarised into profiles/
# (profiles/README.md).
cd "$(dirname "$0")/.."
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
for c in c2 c3 c4; do timeout 400 python bench.py --config $c --steps 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in c3 c4; do timeout 400 python bench.py --sharded --config $c --steps 3 --warmup 2 > $O/bench_sharded1_$c.json 2> $O/bench_sharded1_$c.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/reference_c1.json 2> $O/reference_c1.err
for c in c1 c2 c3 c4; do timeout 300 python tools/profile_step.py --config $c --reps 3 > $O/events_$c.txt 2>&1; done
timeout 300 python tools/gpu/plan_timing.py c1 c2 c3 c4 > $O/plan_timing.txt 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-verify > $O/launches_c1.csv 2> $O/launches_c1.err
NCU="ncu --set full --clock-control none --import-source on"
P="python tools/profile_step.py --reps 1"
timeout 400 $NCU -k regex:zgemm_tma_kernel -s 1 -c 1 -o $O/zgemm_tma_c1 $P --config c1 > /dev/null 2>&1
timeout 400 $NCU -k regex:zgemm_tmap_colm -s 0 -c 1 -o $O/zgemm_tmap_colm_c1 $P --config c1 > /dev/null 2>&1
# blk_level_kernel: c1 has 3 levels per solve (2 warm-up solves + 1): -s 7 = level 1 of the last
timeout 400 $NCU -k regex:blk_level -s 7 -c 1 -o $O/blk_c1_l1 $P --config c1 > /dev/null 2>&1
# c3: 4 levels per solve: level 1 of the last solve; c2: 12 levels: level 5 of the last
timeout 600 $NCU -k regex:blk_level -s 9 -c 1 -o $O/blk_c3_l1 $P --config c3 > /dev/null 2>&1
timeout 600 $NCU -k regex:blk_level -s 29 -c 1 -o $O/blk_c2_l5 $P --config c2 > /dev/null 2>&1
timeout 400 $NCU -k regex:schur_reorder -c 1 -o $O/schur_reorder_c1 python tools/gpu/plan_timing.py c1 > /dev/null 2>&1
timeout 400 $NCU -k regex:block_eig -c 1 -o $O/block_eig_c1 python tools/gpu/plan_timing.py c1 > /dev/null 2>&1
timeout 600 $NCU -k regex:binary_pass -s 1 -c 1 -o $O/binary_pass_c4 $P --config c4 > /dev/null 2>&1
timeout 600 $NCU -k regex:binary_fused -s 1 -c 1 -o $O/binary_fused_c4 $P --config c4 > /dev/null 2>&1
timeout 600 python tools/bench_ode.py > $O/ode_bench.json 2> $O/ode_bench.err
timeout 300 python tools/gpu/route_survey.py > $O/route_survey.txt 2>&1
echo done > $O/done
