timeout 600 python -m pytest tests/test_gpu_accum.py -x -q 2>&1 | tail -2
for v in 2 6 7 8 9 10; do
  echo "variant $v"
  SMX_ACCUM_VARIANT=$v timeout 120 python tools/prof_case.py accum h2d 4096 16 runs 8
  SMX_ACCUM_VARIANT=$v timeout 120 python tools/prof_case.py accum bb 4095 16 runs 8
  SMX_ACCUM_VARIANT=$v timeout 120 python tools/prof_case.py accum h2d 1024 16 runs 8
done
