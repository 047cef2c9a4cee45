timeout 900 python -m pytest tests/test_gpu_ca.py -x -q 2>&1 | tail -2
for c in "h3d 64 4" "h3d 128 8" "h3d 256 8"; do timeout 120 python tools/prof_case.py ca $c bits 6; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_pack_bits|k_unpack_bits" --csv python tools/prof_case.py ca h3d 256 8 bits 3 2>/dev/null | grep -E "k_pack|k_unpack" | head -12
