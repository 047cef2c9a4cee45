timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python bench.py --steps 3 --warmup 3 --no-configs > gpurun_out/launches_raw.csv 2> /dev/null; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pack_bits|k_ca_bits|k_unpack_bits" -s 6 -c 3 -o gpurun_out/c2_full python tools/prof_case.py ca h3d 64 4 runs 4 > /dev/null 2>&1; echo "ncu full rc=$?"
