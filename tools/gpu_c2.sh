timeout 900 python -m pytest tests/test_gpu_ca.py -x -q 2>&1 | tail -2
for c in "h3d 64 4" "bb 63 4" "h3d 128 8"; do timeout 120 python tools/prof_case.py engine $c bits 6 | sed 's/, all=.*//'; done
timeout 600 python bench.py --no-configs > gpurun_out/bench_nc.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_nc.json')); print(d['value'], d['e2e']['value'], d['roofline']['kernel_ms'])"
