set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 2400 python -m pytest tests/ -m gpu -q -x -s ${PYTEST_EXTRA} > gpurun_out/pytest_all.log 2>&1; echo pytest rc $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench rc $?
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench $c rc $?; done
