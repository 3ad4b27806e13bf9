set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests/ -m gpu -q -x > gpurun_out/pytest_full.log 2>&1; echo pytest rc $?
bash tools/refresh_profiles.sh; echo refresh rc $?
