# C2 engine experiment: parity (CA tests), the C2 headline (no config rows), step floor
timeout 900 python -m pytest tests/test_gpu_ca.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('C2', d['value'], d['ms_per_step'], 'bb', d.get('bb'), 'e2e', d['e2e']['value'])"
timeout 300 python tools/step_floor.py 2>&1 | tail -12
