set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -s --deselect "tests/test_gpu_fullsize.py::test_full_config_against_reference_fixture[c3]" --deselect "tests/test_gpu_fullsize.py::test_full_config_against_reference_fixture[c4]" > gpurun_out/pytest1.log 2>&1; echo pytest rc $?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc $?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref1.json 2> gpurun_out/ref1.err; echo ref rc $?
