# single-step CA at C2 (H3D(64) rho=4): per-kernel launch list, full capture of k_ca_fused
timeout 120 python tools/prof_case.py ca h3d 64 4 runs 10 | sed 's/, all=.*//'
timeout 120 python tools/prof_case.py ca h3d 64 4 bits 10 | sed 's/, all=.*//'
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv python tools/prof_case.py ca h3d 64 4 runs 3 > gpurun_out/fusedc2_list.csv 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv python tools/prof_case.py ca h3d 64 4 bits 3 > gpurun_out/bitsc2_list.csv 2>/dev/null
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_ca_fused -s 2 -c 1 -o gpurun_out/fused_c2 python tools/prof_case.py ca h3d 64 4 runs 3 > /dev/null 2>&1
echo done
