timeout 600 python -m pytest tests/test_gpu_accum.py -x -q 2>&1 | tail -1
for a in "h2d 4096 16" "bb 4095 16" "h2d 1024 16"; do timeout 120 python tools/prof_case.py accum $a runs 8 | sed 's/, all=.*//'; done
