timeout 900 python -m pytest tests/test_gpu_ca.py -x -q 2>&1 | tail -3
python tools/prof_case.py ca h3d 256 8 runs 6
python tools/prof_case.py ca h3d 128 8 runs 6
python tools/prof_case.py ca bb 127 8 runs 6
python tools/prof_case.py ca h3d 64 4 runs 6
python tools/prof_case.py ca bb 63 4 runs 6
python tools/prof_case.py ca h3d 16 17 block 6
python tools/prof_case.py ca h3d 64 4 block 6
