set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ode.py -m gpu -q -x > gpurun_out/pytest_bw.log 2>&1; echo pytest rc $?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "c4" > gpurun_out/pytest_bw_full.log 2>&1; echo pytest full rc $?
timeout 300 python tools/profile_step.py --config c4 --reps 3 > gpurun_out/prof_bw_c4.txt 2>&1; echo prof rc $?
