# fixed per-call costs of launch_ca at C2: plan / pack / unpack (ncu full, one launch each)
for k in k_ca_plan k_pack_bits k_unpack_bits; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/fixed_$k python tools/prof_case.py engine h3d 64 4 bits 3 > /dev/null 2>&1; echo "$k $?"
done
