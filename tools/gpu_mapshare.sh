# Issue-slot share of map arithmetic (north star: "issue-slot share spent on map
# arithmetic"): one ncu SourceCounters capture per kernel; tools/map_share.py
# attributes executed instructions to smx_maps.hpp lines here.
set -x
mkdir -p gpurun_out/mapshare
NCU="ncu --section SourceCounters --section LaunchStats --clock-control none --import-source on -c 1"
P="python tools/prof_case.py"
timeout 300 $NCU -k regex:k_map_block -o gpurun_out/mapshare/map_h2d $P map h2d 1024 1 runs 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_map_block -o gpurun_out/mapshare/map_bb2d $P map bb 1023 1 runs 2 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_map_block -o gpurun_out/mapshare/map_h3d $P map h3d 256 1 runs 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_map_block -o gpurun_out/mapshare/map_bb3d $P map bb 255 1 runs 2 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_accum_block -o gpurun_out/mapshare/accum_block_h2d $P accum h2d 1024 16 block 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_accum_block -o gpurun_out/mapshare/accum_block_bb $P accum bb 1023 16 block 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_accum_runs -o gpurun_out/mapshare/accum_runs_h2d $P accum h2d 1024 16 runs 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_accum_runs -o gpurun_out/mapshare/accum_runs_bb $P accum bb 1023 16 runs 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_ca_block -o gpurun_out/mapshare/ca_block_h3d $P ca h3d 64 4 block 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_ca_block -o gpurun_out/mapshare/ca_block_bb $P ca bb 63 4 block 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_ca_plan -o gpurun_out/mapshare/ca_plan_h3d $P engine h3d 64 4 bits 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_ca_bits_run -o gpurun_out/mapshare/ca_run_h3d $P engine h3d 64 4 bits 2 > /dev/null 2>&1
timeout 300 $NCU -k regex:k_edm_runs -o gpurun_out/mapshare/edm_runs_h2d python - > /dev/null 2>&1 <<'PY'
import sys, torch; sys.path.insert(0, '.')
from paper_2208_11617_b200 import api
g = api.make_grid(api.map_kind.h2d, 2, 1024, 16); n = api.tri_cells(g.cell_side())
p = torch.from_numpy(api.make_edm_points(g.cell_side(), 7)).cuda(); e = torch.empty(n, dtype=torch.float64, device='cuda')
api.edm_device(g, p, e, api.EXEC_RUNS); torch.cuda.synchronize()
PY
timeout 300 $NCU -k regex:k_ca2d_runs -o gpurun_out/mapshare/ca2d_runs_h2d $P ca2d h2d 1024 16 runs 2 > /dev/null 2>&1
ls gpurun_out/mapshare
