timeout 2400 python -m pytest tests/ -m gpu -q -x > gpurun_out/s20_pytest.log 2>&1; echo pytest rc $?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s20_smoke.log 2>&1; echo smoke rc $?
bash tools/refresh_profiles.sh; echo refresh rc $?
