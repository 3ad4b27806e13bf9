set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "diagonalised or reduced or cubic or host_path" > gpurun_out/pytest_parity5.log 2>&1; echo pytest rc $?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "c1 or c3" > gpurun_out/pytest_full5.log 2>&1; echo pytest full rc $?
for c in c1 c3; do timeout 300 python tools/profile_step.py --config $c --reps 3 > gpurun_out/prof5_$c.txt 2>&1; echo prof $c rc $?; done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_step.py --config c1 --reps 1 > gpurun_out/launches5_c1.csv 2>/dev/null
timeout 400 ncu --set full --clock-control none --import-source on -k regex:blk_level -s 14 -c 1 -o gpurun_out/blk5_c1_l4 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
