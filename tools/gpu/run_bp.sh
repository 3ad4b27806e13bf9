set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bin or c4 or 2x2 or all_modes" > gpurun_out/pytest_bp.log 2>&1; echo pytest rc $?
timeout 300 python tools/profile_step.py --config c4 --reps 2 > gpurun_out/prof_bp_c4.txt 2>&1; echo prof rc $?
