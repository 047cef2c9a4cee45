# engine change check: CA parity (3-D + 2-D), C2 headline, step floor, C4/C5 engine
timeout 900 python -m pytest tests/test_gpu_ca.py tests/test_gpu_maps2d.py tests/test_gpu_dist.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('C2', d['value'], d['ms_per_step'], 'bb', d.get('bb',{}).get('gcell_steps_s'), 'e2e', d['e2e']['value'])"
timeout 300 python tools/step_floor.py 2>&1 | grep -E "h3d\(4\)|h3d\(64\)|h3d\(128\)"
timeout 120 python tools/prof_case.py engine h3d 256 8 bits 4 | sed 's/, all=.*//'
timeout 120 python tools/prof_case.py engine bb 255 8 bits 4 | sed 's/, all=.*//'
timeout 120 python tools/prof_case.py ca2d h2d 1024 16 runs 6 | sed 's/, all=.*//'
