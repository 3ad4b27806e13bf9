set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ode.py -m gpu -q -x > gpurun_out/pytest_tma.log 2>&1; echo pytest rc $?
timeout 300 python tools/profile_step.py --config c1 --reps 3 > gpurun_out/prof_tma_c1.txt 2>&1; echo prof rc $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_tma_c1.json 2> gpurun_out/bench_tma_c1.err; echo bench rc $?
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_tma_$c.json 2> gpurun_out/bench_tma_$c.err; echo bench $c rc $?; done
