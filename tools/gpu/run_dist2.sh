set -x
timeout 1200 python -m pytest tests/test_distributed.py -m gpu -q -x -s > gpurun_out/pytest_dist.log 2>&1; echo pytest rc $?
NDS_SOLVE_TRACE=1 timeout 300 python tools/profile_step.py --config c1 --reps 1 > gpurun_out/prof_c1.txt 2> gpurun_out/trace_c1.txt; echo trace rc $?
NDS_SOLVE_TRACE=1 timeout 300 python tools/profile_step.py --config c3 --reps 1 > gpurun_out/prof_c3.txt 2> gpurun_out/trace_c3.txt; echo trace rc $?
timeout 600 python bench.py --sharded --config c1 --steps 5 --warmup 2 > gpurun_out/bench_sh_c1.json 2> gpurun_out/bench_sh_c1.err; echo sh c1 rc $?
