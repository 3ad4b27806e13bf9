timeout 2400 python -m pytest tests/ -m gpu -q -x > gpurun_out/s18_pytest.log 2>&1; echo pytest rc $?
bash tools/refresh_profiles.sh; echo refresh rc $?
