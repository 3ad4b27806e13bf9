set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_mbfar.log 2>&1; echo pytest rc $?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "fixture and (c1 or c3)" > gpurun_out/pytest_mbfar_full.log 2>&1; echo pytest full rc $?
for c in c1 c2 c3; do timeout 300 python tools/profile_step.py --config $c --reps 3 > gpurun_out/prof_mbfar_$c.txt 2>&1; echo prof rc $?; done
timeout 300 ncu --set full --clock-control none -k regex:far_group -s 20 -c 1 -o gpurun_out/far_mb_c1 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
