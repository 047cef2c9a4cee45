# A/B of persistent-engine launch shapes (SMX_RUN_VARIANT) at C2 / small grids / C5, plus bare grid.sync cost
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/gsp tools/gridsync_probe.cu && /tmp/gsp
for v in 0 1 3; do
  echo "== variant $v"
  SMX_RUN_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('C2', d['value'], d['ms_per_step'], 'bb', d.get('bb',{}).get('gcell_steps_s'))"
  SMX_RUN_VARIANT=$v timeout 300 python tools/step_floor.py 2>&1 | grep -E "h3d\(4\)|h3d\(32\) rho=4|h3d\(64\)|h3d\(128\)"
  SMX_RUN_VARIANT=$v timeout 120 python tools/prof_case.py engine h3d 256 8 bits 4 | sed 's/, all=.*//'
done
SMX_RUN_VARIANT=1 timeout 900 python -m pytest tests/test_gpu_ca.py -x -q 2>&1 | tail -1
