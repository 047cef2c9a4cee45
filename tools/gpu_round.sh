# Round check on one B200 (regenerates profiles/r2 after tools/ncu_summary.py):
# smoke, GPU tests, default bench, the ncu launch list of the bench, full ncu
# captures of the headline kernel (k_accum_runs, C3) and of the CA engine at
# C5 (k_cols_run), the engine A/B. Outputs: gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -6
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 800 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-configs --no-energy > gpurun_out/launches_raw.csv 2> /dev/null; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_accum_runs" -s 2 -c 1 -o gpurun_out/c3_accum python tools/prof_case.py accum h2d 4096 16 runs 3 > /dev/null 2>&1; echo "ncu full c3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cols_run" -c 1 -o gpurun_out/c5_cols_run python tools/prof_engine.py h3d 256 8 2 > /dev/null 2>&1; echo "ncu full c5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ca2d_runs|pack2d" -s 4 -c 2 -o gpurun_out/f3_ca2d python tools/prof_case.py ca2d h2d 1024 16 runs 4 > /dev/null 2>&1; echo "ncu full f3 rc=$?"
for e in cols chunks; do SMX_CA_ENGINE=$e timeout 300 python tools/engine_ab.py >> gpurun_out/engine_ab.txt 2>&1; done
