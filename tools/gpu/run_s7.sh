set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s7_smoke.log 2>&1; echo smoke rc $?
timeout 2400 python -m pytest tests/ -m gpu -q -x > gpurun_out/s7_pytest.log 2>&1; echo pytest rc $?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s7_bench_c1.json 2> gpurun_out/s7_bench_c1.err; echo bench rc $?
for c in c2 c3; do timeout 400 python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/s7_bench_$c.json 2> gpurun_out/s7_bench_$c.err; echo bench $c rc $?; done
