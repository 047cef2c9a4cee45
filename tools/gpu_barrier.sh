for v in 0 1 2 3; do
  echo "variant $v"
  SMX_BARRIER_VARIANT=$v timeout 300 python tools/step_floor.py 2>&1 | grep -E "h3d\(4\)|h3d\(64\) rho=4|h3d\(128\)"
  SMX_BARRIER_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_ca.py -x -q -k "many_steps or rows_vs" 2>&1 | tail -1
done
