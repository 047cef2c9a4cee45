# The reference's ten-criterion acceptance gate through the GPU path
# (the pool closed compute-sanitizer late in round 2: the sanitizer lines of the
# 12-row column engine and 2-D Life bit-triangle cases stay empty there)
# (tests/acceptance_gpu.py) + compute-sanitizer memcheck / racecheck on small
# cases of every kernel family. Outputs: gpurun_out/acceptance.txt, sanitizer.txt.
python tests/acceptance_gpu.py > gpurun_out/acceptance.txt 2>&1; echo "rc=$?" >> gpurun_out/acceptance.txt
run() {  # env, case
  echo "== memcheck $2 ($1)" >> gpurun_out/sanitizer.txt
  env $1 timeout 300 compute-sanitizer --tool memcheck --leak-check no python tools/prof_case.py $2 2>&1 | grep -E "ERROR SUMMARY|Invalid|Error|failed|No such" | head -5 >> gpurun_out/sanitizer.txt
  echo "== racecheck $2 ($1)" >> gpurun_out/sanitizer.txt
  env $1 timeout 300 compute-sanitizer --tool racecheck python tools/prof_case.py $2 2>&1 | grep -E "RACECHECK SUMMARY|ERROR SUMMARY|hazard|failed|No such" | head -5 >> gpurun_out/sanitizer.txt
}
run SMX_CA_ENGINE=chunks "ca h3d 16 4 runs 2"
run SMX_CA_ENGINE=chunks "ca h3d 16 8 bits 2"
run SMX_CA_ENGINE=chunks "engine h3d 16 4 bits 2"
run SMX_CA_ENGINE=cols "engine h3d 32 8 bits 2"
run SMX_CA_ENGINE=cols "engine bb 31 4 bits 2"
run SMX_CA_ENGINE=auto "multi h3d 32 8 bits 2"
run SMX_CA_ENGINE=auto "accum h2d 64 16 runs 2"
run SMX_CA_ENGINE=auto "kaccum h2d 64 16 runs 2"
run SMX_CA_ENGINE=auto "ca bb 15 4 block 2"
run "SMX_CA_ENGINE=cols SMX_COLS_ROWS=12" "engine h3d 32 8 bits 2"
run "SMX_CA_ENGINE=cols SMX_COLS_ROWS=12" "engine bb 31 4 bits 2"
run "SMX_CA_ENGINE=cols SMX_COLS_ROWS=12" "engine h3d 16 16 bits 2"
run SMX_CA_ENGINE=auto "ca2d h2d 64 16 runs 2"
run SMX_CA_ENGINE=auto "ca2d h2d 64 4 runs 2"
