# Round check on one B200: smoke, GPU tests, default bench, ncu launch list of
# the bench, one full ncu capture of the dominant kernel. Outputs: gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
ls MEASURED_PEAKS.json 2>/dev/null && cat MEASURED_PEAKS.json
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 800 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-configs > gpurun_out/launches_raw.csv 2> /dev/null; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ca_bits_run" -s 1 -c 1 -o gpurun_out/c2_ca_bits_run python bench.py --steps 2 --warmup 3 --no-configs > /dev/null 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ca_bits_run" -s 1 -c 1 -o gpurun_out/c5_ca_bits_run python tools/prof_case.py engine h3d 256 8 bits 2 > /dev/null 2>&1; echo "ncu full c5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_accum_runs" -s 2 -c 1 -o gpurun_out/c3_accum python tools/prof_case.py accum h2d 4096 16 runs 3 > /dev/null 2>&1; echo "ncu full c3 rc=$?"
