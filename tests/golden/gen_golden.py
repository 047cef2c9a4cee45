"""Generate tests/golden/*.json from the REFERENCE ITSELF (oracle/_ref: the
unmodified /root/reference headers compiled in place by oracle/Makefile).

Run in the build container (the only place /root/reference exists):
    make -C oracle && python tests/golden/gen_golden.py
The JSON it writes is committed; the tests never need /root/reference.

Contents
  maps.json   per-grid FNV-1a-64 of the int64 map_outcome array (6 x i64 per block,
              natural z,y,x order) for BB/H2D/H3D; full arrays for tiny grids;
              launch_map counters + exact space_overhead + coverage hash with rho.
  accum.json  launch_accum state hashes (one pass) per (kind, n, rho).
  ca.json     make_life_state hashes and kernel_ca_run / launch_ca final hashes.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import BB, H2D, H3D, Reference, cells_of  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def fnv(arr: np.ndarray) -> int:
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(arr).view(np.uint8).tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def fnv_fast(R: Reference, arr: np.ndarray) -> int:
    # hash of raw bytes through the reference's own FNV (state_hash with m=0, side=0 prefix)
    return R.state_hash(0, 0, arr)


def main() -> None:
    R = Reference()
    t0 = time.time()
    maps = {"hash_note": "state_hash(m=0, side=0, int64 outcome bytes) via the reference's fnv1a",
            "outcomes": [], "tiny": [], "launch_map": []}
    for kind, m, ns in [(H2D, 2, [2, 4, 8, 16, 64, 256, 1024, 4096]),
                        (H3D, 3, [4, 8, 16, 32, 64, 128, 256]),
                        (BB, 2, [1, 2, 7, 63, 1023]),
                        (BB, 3, [1, 4, 7, 63, 255])]:
        for n in ns:
            o = R.map_outcomes(kind, m, n)
            maps["outcomes"].append({"kind": kind, "m": m, "n": n, "blocks": int(o.shape[0]),
                                     "voids": int(o[:, 0].sum()), "hash": fnv_fast(R, o)})
    for kind, m, n in [(H2D, 2, 8), (H3D, 3, 4), (H3D, 3, 8), (BB, 2, 4), (BB, 3, 4)]:
        maps["tiny"].append({"kind": kind, "m": m, "n": n, "outcomes": R.map_outcomes(kind, m, n).tolist()})
    for kind, m, n, rho in [(H2D, 2, 16, 1), (BB, 2, 4, 1), (BB, 3, 4, 1), (H2D, 2, 64, 2), (H2D, 2, 64, 4),
                            (H3D, 3, 8, 2), (BB, 3, 4, 2), (H2D, 2, 1024, 16), (BB, 2, 1023, 16),
                            (H3D, 3, 64, 4), (BB, 3, 63, 4), (H3D, 3, 128, 8), (H3D, 3, 16, 3),
                            (BB, 3, 15, 3), (H2D, 2, 1024, 1), (BB, 2, 1023, 1), (H3D, 3, 256, 1),
                            (BB, 3, 255, 1), (H2D, 2, 32, 5)]:
        cov, cnt = R.launch_map(kind, m, n, rho)
        maps["launch_map"].append({"kind": kind, "m": m, "n": n, "rho": rho,
                                   "blocks_launched": cnt[0], "blocks_void": cnt[1],
                                   "threads_launched": cnt[2], "threads_useful": cnt[3],
                                   "space_overhead": [cnt[4], cnt[5]],
                                   "coverage_hash": fnv_fast(R, cov), "all_one": bool((cov == 1).all())})
    # BB(127) at rho = 8 without coverage (counters only; 1e9 thread iterations)
    _, cnt = R.launch_map(BB, 3, 127, 8, coverage=False)
    maps["launch_map"].append({"kind": BB, "m": 3, "n": 127, "rho": 8, "blocks_launched": cnt[0],
                               "blocks_void": cnt[1], "threads_launched": cnt[2], "threads_useful": cnt[3],
                               "space_overhead": [cnt[4], cnt[5]]})
    json.dump(maps, open(os.path.join(OUT, "maps.json"), "w"), indent=1)
    print("maps", time.time() - t0, flush=True)

    accum = {"launch_accum": []}
    for kind, m, n, rho in [(H2D, 2, 2, 1), (H2D, 2, 16, 1), (H2D, 2, 1024, 1), (H2D, 2, 1024, 16),
                            (BB, 2, 1023, 16), (H2D, 2, 4096, 1), (H2D, 2, 64, 3), (BB, 2, 63, 3),
                            (H2D, 2, 256, 16), (BB, 2, 255, 16), (H2D, 2, 128, 32)]:
        cells, cnt, h, secs = R.launch_accum(kind, m, n, rho, passes=1)
        accum["launch_accum"].append({"kind": kind, "m": m, "n": n, "rho": rho, "hash": h,
                                      "threads_useful": cnt[3], "blocks_void": cnt[1]})
        # two passes: every cell 2
        if n <= 256:
            cells2, _, h2, _ = R.launch_accum(kind, m, n, rho, passes=2)
            accum["launch_accum"][-1]["hash_2pass"] = h2
    json.dump(accum, open(os.path.join(OUT, "accum.json"), "w"), indent=1)
    print("accum", time.time() - t0, flush=True)

    ca = {"life_init": [], "kernel_ca_run": [], "launch_ca": []}
    for m, side, seed in [(3, 7, 11), (3, 15, 42), (3, 63, 42), (3, 255, 42), (3, 1016, 42), (3, 252, 42),
                          (2, 64, 5), (3, 2040, 42)]:
        s = R.make_life_state(m, side, seed)
        ca["life_init"].append({"m": m, "side": side, "seed": seed, "hash": R.state_hash(m, side, s),
                                "alive": int(s.sum())})
    for side, steps, seed in [(6, 1, 0), (7, 6, 11), (15, 64, 42), (31, 64, 42), (63, 4, 42), (63, 64, 42),
                              (63, 100, 42), (127, 8, 42), (255, 1, 42), (255, 2, 42), (31, 64, 0xC0FFEE),
                              (60, 3, 7), (24, 5, 1), (28, 5, 9), (12, 10, 3)]:
        s = R.make_life_state(3, side, seed)
        s, secs = R.kernel_ca_run(3, side, steps, s)
        ca["kernel_ca_run"].append({"side": side, "steps": steps, "seed": seed,
                                    "hash": R.state_hash(3, side, s), "alive": int(s.sum()),
                                    "seconds": round(secs, 3)})
        print("ca", side, steps, secs, flush=True)
    for kind, n, rho, steps in [(H3D, 8, 2, 6), (BB, 7, 2, 6), (H3D, 16, 4, 3), (BB, 15, 4, 3),
                                (H3D, 8, 8, 2), (BB, 7, 8, 2), (H3D, 16, 3, 2)]:
        side = (n - 1 if kind == H3D else n) * rho
        s = R.make_life_state(3, side, 42)
        s, cnt, h, secs = R.launch_ca(kind, 3, n, rho, steps, s)
        ca["launch_ca"].append({"kind": kind, "n": n, "rho": rho, "steps": steps, "seed": 42, "side": side,
                                "hash": h, "blocks_launched": cnt[0], "blocks_void": cnt[1],
                                "threads_useful": cnt[3]})
    json.dump(ca, open(os.path.join(OUT, "ca.json"), "w"), indent=1)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
