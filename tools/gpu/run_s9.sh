set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/s9_parity.log 2>&1; echo pytest rc $?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "c1 or c4" > gpurun_out/s9_full.log 2>&1; echo pytest full rc $?
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s9_bench_c1.json 2> gpurun_out/s9_bench_c1.err; echo bench rc $?
timeout 400 python bench.py --config c4 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/s9_bench_c4.json 2> gpurun_out/s9_bench_c4.err; echo bench c4 rc $?
