timeout 300 compute-sanitizer --tool memcheck python tools/prof_case.py ca h3d 16 4 runs 2 2>&1 | tail -12
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_ca.py -x -q 2>&1 | tail -15
python tools/prof_case.py ca h3d 256 8 runs 6
python tools/prof_case.py ca bb 255 8 runs 6
python tools/prof_case.py engine h3d 256 8 runs 4
python tools/prof_case.py ca h3d 128 8 runs 6
python tools/prof_case.py ca h3d 64 4 runs 6
python tools/prof_case.py ca bb 63 4 runs 6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ca_bits -s 2 -c 1 -o gpurun_out/cab_c5 python tools/prof_case.py ca h3d 256 8 runs 4 > gpurun_out/ncu_cab.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_pack_bits -s 2 -c 1 -o gpurun_out/pack_c5 python tools/prof_case.py ca h3d 256 8 runs 4 > gpurun_out/ncu_pack.log 2>&1
tail -2 gpurun_out/ncu_cab.log
timeout 600 ncu --set full --clock-control none -k regex:k_unpack_bits -s 2 -c 1 -o gpurun_out/unpack_c5 python tools/prof_case.py ca h3d 256 8 runs 4 > gpurun_out/ncu_unpack.log 2>&1
