set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cli.py tests/test_integration.py tests/test_gpu_ode.py -m gpu -q -x > gpurun_out/pytest_e2e.log 2>&1; echo pytest rc $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo bench rc $?
