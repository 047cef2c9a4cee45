# A/B of persistent-engine launch shapes (SMX_RUN_VARIANT) at C2 / small grids
SMX_RUN_VARIANT=1 timeout 900 python -m pytest tests/test_gpu_ca.py -x -q 2>&1 | tail -1
SMX_RUN_VARIANT=2 timeout 900 python -m pytest tests/test_gpu_ca.py -x -q -k "engine or run or launch_ca" 2>&1 | tail -1
for v in 0 1 2; do
  echo "== variant $v"
  SMX_RUN_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('C2', d['value'], d['ms_per_step'], 'bb', d.get('bb',{}).get('gcell_steps_s'), 'e2e', d['e2e']['value'])"
  SMX_RUN_VARIANT=$v timeout 300 python tools/step_floor.py 2>&1 | grep -E "h3d\(4\)|h3d\(32\) rho=4|h3d\(64\) rho=4|bb\(63\)"
done
