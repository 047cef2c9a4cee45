"""Generate tests/golden/maps2d.json from the REFERENCE ITSELF (oracle/_ref:
the unmodified /root/reference headers compiled in place) for the general-n
and comparison 2-D maps: RB, lambda, H padded,
concurrent trapezoids.

    make -C oracle && python tests/golden/gen_golden_2d.py

Contents (hashes are the reference's fnv1a over the raw bytes, state_hash with
m = 0, side = 0):
  outcomes        per grid: blocks, voids, hash of the int64 map_outcome array
                  (6 x i64 per block, the reference's own emission order:
                  detail::for_each_block_outcome, bands one after another)
  decompositions  decompose_trapezoids(n, T) band lists
  launch_map      counters, exact space_overhead, coverage hash, all_one
  launch_accum    one-pass state hash (and threads_useful)
  edm             kernel_edm hashes and launch_edm through maps
  ca2d            2-D periodic Life: make_life_state(2, ...) hashes, kernel_ca_run
                  final hashes, launch_ca through maps
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import BB, H2D, LAMBDA, PADDED, RB, TRAP, Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

OUTCOME_GRIDS = ([(RB, n, 1) for n in (1, 2, 3, 8, 27, 100, 1023, 1024)]
                 + [(LAMBDA, n, 1) for n in (1, 2, 5, 64, 1000)]
                 + [(PADDED, n, 1) for n in (2, 3, 5, 27, 100, 255, 257, 1000, 1025)]
                 + [(TRAP, n, T) for T in (1, 4, 16) for n in (2, 3, 16, 27, 100, 257, 1000, 4095)])
MAP_GRIDS = [(RB, 27, 3, 1), (RB, 1024, 16, 1), (RB, 1023, 16, 1), (LAMBDA, 50, 2, 1), (LAMBDA, 1023, 16, 1),
             (PADDED, 100, 4, 1), (PADDED, 1025, 16, 1), (PADDED, 9, 1, 1), (TRAP, 100, 4, 4), (TRAP, 257, 2, 1),
             (TRAP, 1000, 16, 16), (TRAP, 1000, 16, 1), (TRAP, 27, 5, 4)]
ACCUM_GRIDS = [(RB, 27, 3, 1), (RB, 1024, 16, 1), (LAMBDA, 1023, 16, 1), (PADDED, 1025, 16, 1),
               (PADDED, 100, 3, 1), (TRAP, 1000, 16, 16), (TRAP, 1000, 16, 1), (TRAP, 257, 2, 4),
               (TRAP, 4095, 4, 1)]


def main() -> None:
    R = Reference()
    h = lambda a: R.state_hash(0, 0, a)  # noqa: E731
    out = {"hash_note": "state_hash(m=0, side=0, bytes) via the reference's fnv1a",
           "outcomes": [], "decompositions": [], "launch_map": [], "launch_accum": []}
    for kind, n, T in OUTCOME_GRIDS:
        o = R.map_outcomes(kind, 2, n, T)
        out["outcomes"].append({"kind": kind, "n": n, "T": T, "blocks": int(o.shape[0]),
                                "voids": int(o[:, 0].sum()), "hash": h(o)})
    for n in (16, 27, 100, 1000, 4095, 65535):
        for T in (1, 4, 16):
            out["decompositions"].append({"n": n, "T": T, "bands": R.decompose_trapezoids(n, T)})
    for kind, n, rho, T in MAP_GRIDS:
        cov, cnt = R.launch_map(kind, 2, n, rho, T)
        out["launch_map"].append({"kind": kind, "n": n, "rho": rho, "T": T, "blocks_launched": cnt[0],
                                  "blocks_void": cnt[1], "threads_launched": cnt[2], "threads_useful": cnt[3],
                                  "space_overhead": [cnt[4], cnt[5]], "coverage_hash": h(cov),
                                  "all_one": bool((cov == 1).all())})
    for kind, n, rho, T in ACCUM_GRIDS:
        cells, cnt, hh, _ = R.launch_accum(kind, 2, n, rho, passes=1, T=T)
        out["launch_accum"].append({"kind": kind, "n": n, "rho": rho, "T": T, "hash": hh,
                                    "threads_useful": cnt[3], "blocks_void": cnt[1]})
    out["edm"] = {"kernel_edm": [], "launch_edm": []}
    for side in (14, 15, 63, 255, 1023):
        for seed in (7, 42, 0xC0FFEE):
            _, hh = R.kernel_edm(side, seed)
            out["edm"]["kernel_edm"].append({"side": side, "seed": seed, "hash": hh})
    for kind, n, rho, T in [(BB, 14, 1, 1), (RB, 14, 1, 1), (LAMBDA, 14, 1, 1), (PADDED, 15, 1, 1), (TRAP, 15, 1, 1),
                            (BB, 15, 1, 1), (H2D, 16, 1, 1), (TRAP, 16, 1, 4), (H2D, 64, 4, 1), (BB, 63, 4, 1),
                            (TRAP, 100, 3, 4), (RB, 85, 3, 1), (LAMBDA, 63, 4, 1), (PADDED, 100, 16, 1)]:
        _, cnt, hh = R.launch_edm(kind, n, rho, 7, T)
        out["edm"]["launch_edm"].append({"kind": kind, "n": n, "rho": rho, "T": T, "seed": 7, "hash": hh,
                                         "threads_useful": cnt[3], "blocks_void": cnt[1]})
    out["ca2d"] = {"life_init": [], "kernel_ca_run": [], "launch_ca": []}
    for side, seed in [(24, 42), (15, 9), (63, 42), (1023, 42), (252, 5)]:
        st = R.make_life_state(2, side, seed)
        out["ca2d"]["life_init"].append({"side": side, "seed": seed, "hash": R.state_hash(2, side, st),
                                         "alive": int(st.sum())})
    for side, steps, seed in [(24, 8, 42), (15, 6, 9), (63, 64, 42), (255, 64, 42), (1023, 64, 42), (255, 64, 0xC0FFEE)]:
        st = R.make_life_state(2, side, seed)
        R.kernel_ca_run(2, side, steps, st)
        out["ca2d"]["kernel_ca_run"].append({"side": side, "steps": steps, "seed": seed,
                                             "hash": R.state_hash(2, side, st)})
    for kind, n, rho, T, steps in [(BB, 24, 1, 1, 8), (RB, 24, 1, 1, 8), (LAMBDA, 24, 1, 1, 8), (TRAP, 25, 1, 1, 8),
                                   (PADDED, 25, 1, 1, 8), (H2D, 16, 1, 1, 6), (TRAP, 16, 1, 4, 6),
                                   (H2D, 64, 4, 1, 5), (BB, 63, 4, 1, 5), (TRAP, 100, 3, 4, 5), (RB, 85, 3, 1, 5)]:
        side = (n - 1 if kind in (H2D, TRAP, PADDED) else n) * rho
        st = R.make_life_state(2, side, 42)
        st, cnt, hh, _ = R.launch_ca(kind, 2, n, rho, steps, st, T=T)
        out["ca2d"]["launch_ca"].append({"kind": kind, "n": n, "rho": rho, "T": T, "steps": steps, "seed": 42,
                                         "side": side, "hash": hh, "threads_useful": cnt[3]})
    json.dump(out, open(os.path.join(OUT, "maps2d.json"), "w"), indent=1)
    print("wrote", os.path.join(OUT, "maps2d.json"))


if __name__ == "__main__":
    main()
