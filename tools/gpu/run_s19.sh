timeout 2400 python -m pytest tests/ -m gpu -q -x > gpurun_out/s19_pytest.log 2>&1; echo pytest rc $?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s19_smoke.log 2>&1; echo smoke rc $?
bash tools/refresh_profiles.sh; echo refresh rc $?
