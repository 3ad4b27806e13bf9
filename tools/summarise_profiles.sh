#!/bin/bash
# Copies what tools/refresh_profiles.sh brought back in gpurun_out/prof/ into profiles/ under the
# round's prefix (default r02): bench lines, event timelines, the c1 launch list and its shares,
# and the `ncu --page details --csv` summary of every .ncu-rep capture.
cd "$(dirname "$0")/.."
R=${1:-r02}
I=gpurun_out/prof
for c in c1 c2 c3 c4; do
  tail -n 1 $I/bench_$c.json > profiles/${R}_bench_$c.json
  cp $I/events_$c.txt profiles/${R}_events_$c.txt
done
for c in c3 c4; do tail -n 1 $I/bench_sharded1_$c.json > profiles/${R}_bench_sharded1_$c.json; done
tail -n 1 $I/reference_c1.json > profiles/${R}_reference_c1.json
cp $I/ode_bench.json profiles/${R}_ode_bench.json  # two lines: OdePropagator::at on c1, RK4 on c0
cp $I/plan_timing.txt profiles/${R}_plan_timing.txt
cp $I/route_survey.txt profiles/${R}_route_survey.txt
cp $I/gpu.txt profiles/${R}_gpu.txt
cp $I/lscpu.txt profiles/${R}_lscpu.txt
grep -v '^==' $I/launches_c1.csv > profiles/${R}_ncu_launches_c1.csv
python tools/launch_shares.py profiles/${R}_ncu_launches_c1.csv > profiles/${R}_launch_shares_c1.txt
for rep in $I/*.ncu-rep; do
  n=$(basename $rep .ncu-rep)
  ncu -i $rep --page details --csv > profiles/${R}_ncu_${n}_details.csv 2>/dev/null
done
ls -la profiles/${R}_*
