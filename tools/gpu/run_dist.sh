set -x
timeout 1200 python -m pytest tests/test_distributed.py -m gpu -q -x -s > gpurun_out/pytest_dist.log 2>&1; echo pytest rc $?
timeout 600 python bench.py --sharded --config c3 --steps 3 --warmup 2 > gpurun_out/bench_sh_c3.json 2> gpurun_out/bench_sh_c3.err; echo sh c3 rc $?
timeout 600 python bench.py --sharded --config c4 --steps 3 --warmup 2 > gpurun_out/bench_sh_c4.json 2> gpurun_out/bench_sh_c4.err; echo sh c4 rc $?
timeout 600 python bench.py --sharded --config c1 --steps 5 --warmup 2 > gpurun_out/bench_sh_c1.json 2> gpurun_out/bench_sh_c1.err; echo sh c1 rc $?
