set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "binary or bin or c4 or 2x2" > gpurun_out/pytest_bs.log 2>&1; echo pytest rc $?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "c4 or c1" > gpurun_out/pytest_bs_full.log 2>&1; echo pytest full rc $?
timeout 300 python tools/profile_step.py --config c1 --reps 3 > gpurun_out/prof_bs_c1.txt 2>&1; echo prof rc $?
timeout 300 python tools/profile_step.py --config c4 --reps 2 > gpurun_out/prof_bs_c4.txt 2>&1; echo prof rc $?
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_bs_c4.json 2> gpurun_out/bench_bs_c4.err; echo bench c4 rc $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_bs_c1.json 2> gpurun_out/bench_bs_c1.err; echo bench c1 rc $?
