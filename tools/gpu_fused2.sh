set -x
timeout 900 python -m pytest tests/test_gpu_ca.py -x -q 2>&1 | tail -4
for c in "h3d 64 4" "bb 63 4" "h3d 128 8" "h3d 256 8" "bb 255 8"; do
  timeout 120 python tools/prof_case.py ca $c runs 8
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ca_fused" -s 2 -c 1 -o gpurun_out/fused2_c5 python tools/prof_case.py ca h3d 256 8 runs 3 > /dev/null 2>&1; echo "ncu rc=$?"
