python tests/acceptance_gpu.py > gpurun_out/acceptance.txt 2>&1; echo "rc=$?" >> gpurun_out/acceptance.txt
for c in "ca h3d 16 4 runs 2" "ca h3d 16 8 bits 2" "engine h3d 16 4 bits 2" "accum h2d 64 16 runs 2" "ca bb 15 4 block 2"; do
  echo "== memcheck $c" >> gpurun_out/sanitizer.txt
  timeout 300 compute-sanitizer --tool memcheck --leak-check no python tools/prof_case.py $c 2>&1 | grep -E "ERROR SUMMARY|Invalid|Error" | head -5 >> gpurun_out/sanitizer.txt
  echo "== racecheck $c" >> gpurun_out/sanitizer.txt
  timeout 300 compute-sanitizer --tool racecheck python tools/prof_case.py $c 2>&1 | grep -E "RACECHECK SUMMARY|ERROR SUMMARY|hazard" | head -5 >> gpurun_out/sanitizer.txt
done
python - >> gpurun_out/sanitizer.txt 2>&1 <<'PY'
PY
