python tools/prof_case.py ca h3d 256 8 runs 6
python tools/prof_case.py ca bb 255 8 runs 6
python tools/prof_case.py ca h3d 64 4 runs 6
python tools/prof_case.py accum h2d 4096 16 runs 6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ca_runs -s 2 -c 1 -o gpurun_out/ca_c5 python tools/prof_case.py ca h3d 256 8 runs 4 > gpurun_out/ncu_ca.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_accum_runs -s 2 -c 1 -o gpurun_out/acc_c3 python tools/prof_case.py accum h2d 4096 16 runs 4 > gpurun_out/ncu_acc.log 2>&1
tail -3 gpurun_out/ncu_ca.log gpurun_out/ncu_acc.log
