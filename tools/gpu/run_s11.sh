timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "superblocks or inner_modes" > gpurun_out/s11_newtests.log 2>&1; echo newtests rc $?
bash tools/refresh_profiles.sh; echo refresh rc $?
