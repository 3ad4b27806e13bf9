set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_parity.log 2>&1; echo pytest rc $?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "c4" > gpurun_out/pytest_full_c4.log 2>&1; echo pytest full rc $?
for c in c1 c2 c3 c4; do timeout 300 python tools/profile_step.py --config $c --reps 3 > gpurun_out/prof_$c.txt 2>&1; echo prof $c rc $?; done
timeout 600 python bench.py --config c4 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench c4 rc $?
