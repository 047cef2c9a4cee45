"""GPU parity of the column engine's two item shapes (8-row `k_cols_run`,
12-row `k_cols_run12`) forced on small states whose sides leave partial row
bands, word groups and z runs (the automatic choice takes 12-row items only at
C5 sizes): launch_ca through the bit-shadow path, H3D and BB, rho 4 / 8 / 16,
against the restated oracle (oracle/smx_oracle.c; the reference's
kernel_ca_run, simulator.hpp:402-425). The shape and the engine are process-
wide settings read once, so each shape runs in a child process."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
from oracle.oracle import Restated
from paper_2208_11617_b200 import api
orc = Restated()
out = []
for kind, n, rho, steps in json.loads(sys.argv[2]):
    g = api.make_grid(api.map_kind[kind], 3, n, rho)
    side = g.cell_side()
    want = orc.make_life_state(3, side, 11)
    orc.ca3d_run(side, steps, want)
    st = api.make_life_state(3, side, 11)
    api.launch_ca(g, api.simplex_spec(3, side - 1), st,
                  api.launch_opts(steps=steps, boundary=api.ca_boundary.dead3d, exec=api.EXEC_BITS,
                                  record_coverage=False))
    out.append([kind, n, rho, side, steps, bool((st.cells == want).all())])
print(json.dumps(out))
"""

# (kind, n, rho, steps): sides 60, 124, 248, 504, 372, 496, 496 and 1016 (C4, one step); all but
# 504 end on a partial 12-row band, 60 and 124 also on a partial 8-row band
CASES = [("h3d", 16, 4, 3), ("h3d", 32, 4, 5), ("h3d", 32, 8, 5), ("bb", 63, 8, 4), ("bb", 93, 4, 3),
         ("h3d", 32, 16, 3), ("bb", 31, 16, 2), ("h3d", 128, 8, 1)]


@pytest.mark.parametrize("rows", [8, 12])
def test_column_engine_shape_vs_oracle(cuda, rows):
    env = dict(os.environ, SMX_CA_ENGINE="cols", SMX_COLS_ROWS=str(rows))
    res = subprocess.run([sys.executable, "-c", CHILD, ROOT, json.dumps(CASES)], env=env, capture_output=True,
                         text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    assert len(got) == len(CASES)
    bad = [r for r in got if not r[-1]]
    assert not bad, f"{rows}-row column engine differs from the oracle: {bad}"
