set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_diag.log 2>&1; echo pytest rc $?
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_cli.py tests/test_gpu_ode.py tests/test_integration.py -m gpu -q -x -k "c4 or cli or ode or integration or dropin or bin" > gpurun_out/pytest_diag_full.log 2>&1; echo pytest full rc $?
timeout 300 python tools/profile_step.py --config c4 --reps 3 > gpurun_out/prof_diag_c4.txt 2>&1; echo prof rc $?
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_diag_c4.json 2> gpurun_out/bench_diag_c4.err; echo bench rc $?
