"""Full-size CA goldens for the bench's self-check and the slow GPU parity
tests: final state hashes of the dead-boundary 3-D Life at the BASELINE
configs' exact (side, steps) tuples, computed by the RESTATED oracle
(oracle/smx_oracle.c, multithreaded row sweep), which tests/test_oracle.py pins
bit-exact against the reference's own kernel_ca_run (sides 15..255, Appendix A)
and which reproduces the reference's side-1023 one-step hash
13036985295180606544 (checked below before anything is
written). The reference itself would need ~20 h for C4 x 100.

    make -C oracle && python tests/golden/gen_golden_full.py      (~3 min on 8 cores)

Writes tests/golden/ca_full.json (committed). Test infrastructure only.
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Restated  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ca_full.json")
SEED = 42

# (label, side, steps, grid note) — the state is map-independent: H3D(n_b) and
# BB(n_b - 1) at the same rho cover the same side
CASES = [
    ("c2_rho4_100", 252, 100, "C2: grid_h3d(64) / grid_bb(63,3), rho=4"),
    ("c4_rho8_100", 1016, 100, "C4: grid_h3d(128) / grid_bb(127,3), rho=8"),
    ("c4_rho8_1", 1016, 1, "C4: one step"),
    ("c5_rho8_2", 2040, 2, "C5: grid_h3d(256) / grid_bb(255,3), rho=8, 2 steps"),
    ("c5_rho8_20", 2040, 20, "C5: 20 steps (the bench's engine call)"),
    ("c5_rho4_20", 2044, 20, "C5 at rho=4: grid_h3d(512), 20 steps"),
    ("c5_rho16_20", 2032, 20, "C5 at rho=16: grid_h3d(128) / grid_bb(127,3), 20 steps"),
    ("side1023_1", 1023, 1, "SURVEY Appendix A: H3D(1024) rho=1 / BB(1023), one step"),
]
APPENDIX_A_1023 = 13036985295180606544


def main() -> None:
    """`python gen_golden_full.py [label ...]`: (re)compute only those cases,
    keeping the others already in ca_full.json."""
    o = Restated()
    out = {"note": __doc__.strip().splitlines()[0], "seed": SEED, "cases": {}}
    only = set(sys.argv[1:])
    if only and os.path.exists(OUT):
        out = json.load(open(OUT))
    for label, side, steps, note in CASES:
        if only and label not in only and label != "side1023_1":
            continue
        t0 = time.time()
        s = o.make_life_state(3, side, SEED)
        init_hash = o.state_hash(3, side, s)
        o.ca3d_run(side, steps, s)
        h = o.state_hash(3, side, s)
        if label == "side1023_1" and h != APPENDIX_A_1023:
            raise SystemExit(f"restated oracle disagrees with the reference at side 1023: {h}")
        out["cases"][label] = {"side": side, "steps": steps, "cells": int(s.size), "init_hash": str(init_hash),
                               "final_hash": str(h), "alive": int(s.sum()), "grid": note}
        print(label, side, steps, h, f"{time.time() - t0:.1f}s", flush=True)
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
