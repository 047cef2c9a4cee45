"""Issue-slot share of map arithmetic per kernel, from ncu SourceCounters captures
(tools/gpu_mapshare.sh -> gpurun_out/mapshare/*.ncu-rep).

Every executed SASS instruction is attributed to its (innermost, -lineinfo)
source line; lines are classed as
  map         the block -> tile arithmetic: include/smx_maps.hpp (map_h2d/h3d/
              bb/..., incl. BB's Void test), map_raw/map_block (smx_common.cuh)
              and the per-warp evaluate-and-broadcast (warp_map, smx_kernels.cu);
  membership  the sweep's per-thread tri/tet_contains filter (simulator.hpp:
              205-207), told apart from map_bb's use by the inline chain;
  chain  map-driven work assembly of the x-run schemes: strip_runs
         (smx_runs.cuh) and build_chunks (smx_ca_common.cuh);
  work   everything else (the workload body, address math, stores).
Also prints the launched-vs-useful block fraction the reports carry.

    python tools/map_share.py [gpurun_out/mapshare] > profiles/r1/map_issue_share.json
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2208_11617_b200", "libsmx_b200.so")


def frames(txt):
    """'//## File "a", line 1 inlined at "b", line 2 ...' -> [(a, 1), (b, 2), ...], innermost first"""
    return [(os.path.basename(f), int(n)) for f, n in re.findall(r'"([^"]+)", line (\d+)', txt)]


def line_map(so, fn):
    """SASS offset -> inline chain of (file, line), for the function named fn"""
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, check=True, capture_output=True)
    for f in sorted(os.listdir(tmp)):
        if not f.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "--print-line-info-inline", "-c", os.path.join(tmp, f)],
                             capture_output=True, text=True).stdout
        # the //## lines before an instruction spell its inline chain, innermost
        # first; an instruction with none keeps the previous chain
        out, cur, fresh, inside = {}, [], True, False
        for ln in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                inside = m.group(1) == fn
                continue
            if "//##" in ln:
                if fresh:
                    cur, fresh = [], False
                cur += [f for f in frames(ln) if f not in cur]
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m:
                fresh = True
                if inside:
                    out[int(m.group(1), 16)] = cur
        if out:
            return out
    return {}


MAPS_CONTAINS = range(69, 76)  # tri_contains / tet_contains in include/smx_maps.hpp


def klass(chain):
    if not chain:
        return "work"
    f, ln = chain[0]
    if f == "smx_maps.hpp":
        if ln in MAPS_CONTAINS and not any(g == "smx_maps.hpp" for g, _ in chain[1:]):
            return "membership"  # the sweep's per-thread filter, not the map (BB's Void test is map_bb's)
        return "map"
    for g, n in chain:
        if (g == "smx_common.cuh" and 33 <= n <= 48) or (g == "smx_kernels.cu" and 42 <= n <= 55):
            return "map"
    if any(g == "smx_runs.cuh" or (g == "smx_ca_common.cuh" and 84 <= n <= 141) for g, n in chain):
        return "chain"
    return "work"


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def mangled(rep):
    rows = ncu_csv(rep, "--page", "raw", "--print-kernel-base", "mangled", "--metrics",
                   "launch__grid_size,smsp__inst_executed.sum")
    h = rows[0]
    r = rows[2] if len(rows) > 2 and rows[1][0] == "" else rows[1]
    return r[h.index("Kernel Name")], float(r[h.index("smsp__inst_executed.sum")].replace(",", "") or 0)


def share(rep):
    name, inst_total = mangled(rep)
    rows = ncu_csv(rep, "--page", "source")
    hi = [i for i, r in enumerate(rows) if "Address" in r][0]
    h = rows[hi]
    ia, ie = h.index("Address"), h.index("Instructions Executed")
    lm = line_map(SO, name)
    body = [r for r in rows[hi + 1:] if len(r) > ie and r[ia]]
    base = min(int(r[ia], 16) for r in body)
    by = collections.Counter()
    unmapped = 0.0
    for r in body:
        v = float(r[ie] or 0)
        chain = lm.get(int(r[ia], 16) - base)
        if chain is None:
            unmapped += v
        by[klass(chain)] += v
    tot = sum(by.values()) or 1.0
    return {
        "kernel": name,
        "warp_inst": tot,
        "map_share": round(by["map"] / tot, 4),
        "membership_share": round(by["membership"] / tot, 4),
        "chain_share": round(by["chain"] / tot, 4),
        "work_share": round(by["work"] / tot, 4),
        "unmapped_share": round(unmapped / tot, 4),
    }


def main():
    d = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "mapshare")
    out = {"source": "ncu --section SourceCounters (tools/gpu_mapshare.sh), SASS -> source lines via -lineinfo "
                     "(tools/map_share.py); share of executed warp instructions",
           "kernels": {}}
    for f in sorted(os.listdir(d)):
        if f.endswith(".ncu-rep"):
            out["kernels"][f[:-8]] = share(os.path.join(d, f))
    # launched vs useful blocks of the profiled grids, from the reference's own
    # launch_map counters (oracle/_ref; this container only)
    try:
        sys.path.insert(0, ROOT)
        from oracle.oracle import BB, H2D, H3D, Reference
        ref = Reference()
        cases = {"map_h2d": (H2D, 2, 1024, 1), "map_bb2d": (BB, 2, 1023, 1), "map_h3d": (H3D, 3, 256, 1),
                 "map_bb3d": (BB, 3, 255, 1), "accum_h2d_rho16": (H2D, 2, 1024, 16),
                 "accum_bb_rho16": (BB, 2, 1023, 16), "ca_h3d_rho4": (H3D, 3, 64, 4), "ca_bb_rho4": (BB, 3, 63, 4)}
        out["blocks"] = {}
        for k, (kind, m, n, rho) in cases.items():
            _, c = ref.launch_map(kind, m, n, rho, coverage=False)
            out["blocks"][k] = {"launched": c[0], "void": c[1], "useful_block_frac": round(1 - c[1] / c[0], 4),
                                "useful_thread_frac": round(c[3] / c[2], 4)}
        out["blocks_source"] = "reference launch_map counters (oracle/_ref, simulator.hpp:303-310)"
    except Exception as e:  # noqa: BLE001 - the reference is absent on the GPU box
        out["blocks"] = f"unavailable: {e}"
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
