"""Attribute ncu per-SASS-instruction metrics to CUDA source lines.

    ncu -i rep.ncu-rep --page source --csv > src.csv
    python tools/sass_lines.py src.csv <kernel-substring> [lib.so]

Maps SASS addresses to file:line with nvdisasm --print-line-info on the cubin
embedded in libsmx_b200.so (built with -lineinfo).
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line_map(so, kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, check=True, capture_output=True)
    out = {}
    for f in sorted(os.listdir(tmp), key=len):
        if not f.endswith(".cubin") or out:
            continue
        txt = subprocess.run(["nvdisasm", "--print-line-info", "-c", os.path.join(tmp, f)],
                             capture_output=True, text=True).stdout
        fn, cur = None, None
        for ln in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                fn = m.group(1)
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and fn and kernel_sub in fn:
                out[int(m.group(1), 16)] = cur
    return out


def main():
    src, ksub = sys.argv[1], sys.argv[2]
    so = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "paper_2208_11617_b200", "libsmx_b200.so")
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if "Address" in r][0]
    h = rows[hi]
    ia, ie, ist = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    lm = line_map(so, ksub)
    inst, stall = collections.Counter(), collections.Counter()
    tot = 0.0
    base = min(int(r[ia], 16) for r in rows[hi + 1:] if len(r) > ie)
    for r in rows[hi + 1:]:
        if len(r) <= ie:
            continue
        a = int(r[ia], 16) - base
        key = lm.get(a, "?")
        v = float(r[ie] or 0)
        inst[key] += v
        stall[key] += float(r[ist] or 0)
        tot += v
    st = sum(stall.values()) or 1
    for k, v in inst.most_common(int(os.environ.get("TOPN", "40"))):
        print(f"{100 * v / tot:6.2f}% inst  {100 * stall[k] / st:6.2f}% stall  {k}")


if __name__ == "__main__":
    main()
