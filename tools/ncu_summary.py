"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU).

    python tools/ncu_summary.py report <name>.ncu-rep [...]   -> markdown rows + JSON
    python tools/ncu_summary.py launches launches_raw.csv     -> per-kernel launch table
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_bytes.sum": "l2_bytes",
}


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {"kernel": v[head.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in head:
                i = head.index(k)
                x = v[i]
                if name.startswith("dram_r") or name.startswith("dram_w") or name == "l2_bytes":
                    d[name] = to_bytes(x, units[i])
                else:
                    try:
                        d[name] = float(x)
                    except ValueError:
                        d[name] = x
        out.append(d)
    return out


def launches(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    ik, im, iu, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    iid = h.index("ID")
    by = {}
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        d = by.setdefault(r[iid], {"kernel": r[ik]})
        val = r[iv].replace(",", "")
        d[r[im]] = to_bytes(val, r[iu]) if r[im].startswith("dram") else float(val)
    return list(by.values())


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "report":
        res = {p: report(p) for p in sys.argv[2:]}
        print(json.dumps(res, indent=1))
    else:
        res = launches(sys.argv[2])
        print(json.dumps(res, indent=1))
