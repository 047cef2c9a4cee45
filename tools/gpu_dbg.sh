CUDA_LAUNCH_BLOCKING=1 timeout 300 compute-sanitizer --tool memcheck python tools/prof_case.py ca h3d 16 4 runs 2 > gpurun_out/san.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 300 compute-sanitizer --tool memcheck python tools/prof_case.py ca h3d 32 8 runs 2 > gpurun_out/san8.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 300 compute-sanitizer --tool memcheck python tools/prof_case.py engine bb 31 8 runs 2 > gpurun_out/san9.log 2>&1
