set -x
O=gpurun_out/s3; mkdir -p $O
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_step.py --config c1 --reps 1 > $O/launches_c1.csv 2> $O/launches_c1.err
timeout 400 ncu --set full --clock-control none --import-source on -k regex:tile_diag_div -s 1 -c 1 -o $O/div_c1_l1 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:tile_diag_div -s 22 -c 1 -o $O/div_c1_l22 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:far_group -s 20 -c 1 -o $O/far_c1_l22 python tools/profile_step.py --config c1 --reps 1 > /dev/null 2>&1
