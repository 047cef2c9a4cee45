# staged-row 2-D Life kernel: parity + timing
timeout 900 python -m pytest tests/test_gpu_maps2d.py -x -q -k ca2d 2>&1 | tail -3
for c in "h2d 1024 16" "bb 1023 16" "h2d 4096 16" "h2d 2048 8" "bb 2047 8" "h2d 512 32"; do timeout 120 python tools/prof_case.py ca2d $c runs 6 | sed 's/, all=.*//'; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_ca2d_rows -s 2 -c 1 -o gpurun_out/ca2d_rows python tools/prof_case.py ca2d h2d 1024 16 runs 3 > /dev/null 2>&1; echo ncu $?
