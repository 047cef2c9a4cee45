# parallel chunk builder: parity of every CA path + per-call fixed costs
timeout 900 python -m pytest tests/test_gpu_ca.py tests/test_gpu_dist.py tests/test_gpu_edges.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('C2', d['value'], d['ms_per_step'], 'bb', d.get('bb',{}).get('gcell_steps_s'), 'e2e', d['e2e']['value'])"
for c in "h3d 64 4 runs" "h3d 64 4 bits" "bb 63 4 runs" "h3d 128 8 runs" "h3d 256 8 bits"; do timeout 120 python tools/prof_case.py ca $c 8 | sed 's/, all=.*//'; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_case.py engine h3d 64 4 bits 3 2>/dev/null | grep -E "k_ca_plan|k_pack|k_unpack|k_ca_bits_run" | head -8 | cut -d, -f5,13-
