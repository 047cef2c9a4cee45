CUDA_LAUNCH_BLOCKING=1 timeout 300 compute-sanitizer --tool memcheck python tools/prof_case.py ca h3d 16 4 runs 2 2>&1 | head -60
