# rho = 4 engine shapes at larger sizes: variant 2 (1 chunk/item, z-split) vs 3 (2 chunks/item)
for v in 2 3; do
  for c in "h3d 128 4" "h3d 256 4" "h3d 512 4"; do SMX_RUN_VARIANT=$v timeout 120 python tools/prof_case.py engine $c bits 4 | sed "s/, all=.*//;s/^/v$v /"; done
done
