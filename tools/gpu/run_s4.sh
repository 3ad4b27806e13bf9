set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "diagonalised or reduced or cubic or host_path" > gpurun_out/pytest_parity4.log 2>&1; echo pytest rc $?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "c1 or c3" > gpurun_out/pytest_full4.log 2>&1; echo pytest full rc $?
for c in c1 c3; do timeout 300 python tools/profile_step.py --config $c --reps 3 > gpurun_out/prof4_$c.txt 2>&1; echo prof $c rc $?; done
NDS_SOLVE_TRACE=1 timeout 300 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2> gpurun_out/trace4_c1.txt
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_step.py --config c1 --reps 1 > gpurun_out/launches4_c1.csv 2>/dev/null
