set -x
timeout 900 python -m pytest tests/test_gpu_ca.py -x -q 2>&1 | tail -4
for c in "h3d 64 4" "bb 63 4" "h3d 128 8" "bb 127 8" "h3d 256 8" "bb 255 8"; do
  timeout 120 python tools/prof_case.py engine $c bits 4
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ca_bits_run" -s 1 -c 1 -o gpurun_out/c2_run python tools/prof_case.py engine h3d 64 4 bits 2 > /dev/null 2>&1; echo "ncu rc=$?"
