set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_pair.log 2>&1; echo pytest rc $?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "fixture and (c1 or c2 or c3)" > gpurun_out/pytest_pair_full.log 2>&1; echo pytest full rc $?
for c in c1 c2 c3; do timeout 300 python tools/profile_step.py --config $c --reps 3 > gpurun_out/prof_pair_$c.txt 2>&1; echo prof rc $?; done
NDS_SOLVE_TRACE=1 timeout 300 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2> gpurun_out/trace_pair_c1.txt
NDS_SOLVE_TRACE=1 timeout 300 python tools/profile_step.py --config c3 --reps 1 > /dev/null 2> gpurun_out/trace_pair_c3.txt
