"""Benchmark driver (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2]

Workload (BASELINE.json configs[1], "C2"): one dead-boundary 3-D Life step over
the voxelised tetrahedron of side 252 through the H3D block-space map
(grid_h3d(64), rho = 4: 2,699,004 u8 cells, seed 42). A bench "step" is one
CA step; `value` is Gcells/s (useful cells x steps / device time), inputs
resident in HBM, L2 flushed (256 MiB write) before every timed step because the
2.7 MB state would otherwise sit in the 126 MB L2. `e2e` is the same step through
the reference-facing C ABI with host (pinned) buffers: H2D + step + D2H per step.

Also reported, per BASELINE config (C1, C3, C4, C5 at 1 GPU): H and BB Gcells/s,
H-vs-BB speedup, HBM roofline fraction, J/cell from NVML, and the paper's MAP
kernel block rate. Multi-GPU (torchrun, N > 1): the CA is sharded over whole H
levels (paper_2208_11617_b200/dist.py) with a tile halo exchange; `value` is the
whole-domain throughput (strong scaling).

`--impl reference` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference headers compiled in place) on the same
workload, one replica per host core.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 42
WORKLOADS = {
    # name: (description, kind, n, rho) for the H grid; BB uses (n-1) for h kinds
    "c2": ("3-simplex n=256 CA step (C2): H3D(64) rho=4, side 252", "h3d", 64, 4),
}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel_key: str):
    """dram bytes per launch for the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        v = d.get(kernel_key, {}).get("dram_bytes_per_launch")
        return float(v) if v is not None else None
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle-reason sampling through NVML."""

    def __init__(self, index=0, period=0.05):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def energy_mj(self):
        if not self.ok:
            return None
        try:
            return self.N.nvmlDeviceGetTotalEnergyConsumption(self.h)
        except Exception:
            return None

    def _run(self):
        N = self.N
        names = {
            "hw_slowdown": getattr(N, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(N, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(N, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def timed_steps(fn, iters, flush=None, stream=None):
    """Per-step CUDA-event timing on the launching (current) stream; the L2
    flush runs between timed steps, outside the events. Returns ms list."""
    import torch
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(iters)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(iters)]
    for i in range(iters):
        if flush is not None:
            flush()
        starts[i].record()
        fn(i)
        ends[i].record()
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)]


class Flusher:
    def __init__(self, mib=256):
        import torch
        self.buf = torch.empty(mib << 20, dtype=torch.uint8, device="cuda")

    def __call__(self):
        self.buf.fill_(1)


def ca_case(api, kind, n, rho, steps, warmup, flush, exec_=None):
    """Time `steps` CA steps (u8 state -> u8 state) on grid (kind, n, rho).
    x-run scheme: the three stages smx_ca_step chains (pack -> bit-sliced step ->
    unpack) are timed individually with events on the launching stream; the
    step time is pack-start to unpack-end. Block scheme: one kernel."""
    import torch
    g = api.make_grid(api.map_kind[kind], 3, n, rho)
    side = g.cell_side()
    cells = api.tet_cells(side)
    a = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
    b = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
    api.life_init_device(3, side, SEED, a)
    ex = api.EXEC_RUNS if exec_ is None else exec_
    bufs = [a, b]
    res = {"grid": f"{kind}({n}) rho={rho}", "side": side, "cells": cells, "g": g, "bufs": bufs}
    if ex == api.EXEC_BLOCK:
        def step(i):
            api.ca_step_device(g, bufs[i % 2], bufs[(i + 1) % 2], ex)

        timed_steps(step, warmup, flush)
        res["ms"] = timed_steps(step, steps, flush)
        res["step"] = step
        return res
    sa, sb = api.bits_buffer(g), api.bits_buffer(g)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]

    def step(i, e=None):
        cur, nxt = bufs[i % 2], bufs[(i + 1) % 2]
        if e: e[0].record()
        api.bits_pack_device(g, cur, sa)
        if e: e[1].record()
        api.bits_step_device(g, sa, sb)
        if e: e[2].record()
        api.bits_unpack_device(g, sb, nxt)
        if e: e[3].record()

    for i in range(warmup):
        flush()
        step(i)
    for i in range(steps):
        flush()
        step(i, ev[i])
    torch.cuda.synchronize()
    res["stage_ms"] = {name: statistics.mean(e[k].elapsed_time(e[k + 1]) for e in ev)
                       for k, name in enumerate(("pack", "step", "unpack"))}

    # the step itself: ONE smx_ca_step call (the library launches the three
    # kernels back to back; per-stage events above would add host gaps)
    def abi_step(i):
        api.ca_step_device(g, bufs[i % 2], bufs[(i + 1) % 2], api.EXEC_RUNS)

    timed_steps(abi_step, warmup, flush)
    res["ms"] = timed_steps(abi_step, steps, flush)
    res["step"] = abi_step

    # multi-step engine (smx_ca): the bit shadow carries over, so a step is
    # step + unpack (the u8 state is still written every step)
    def estep(i):
        src, dst = (sa, sb) if i % 2 == 0 else (sb, sa)
        api.bits_step_device(g, src, dst)
        api.bits_unpack_device(g, dst, bufs[(i + 1) % 2])

    api.bits_pack_device(g, a, sa)
    timed_steps(estep, 2, flush)
    api.bits_pack_device(g, a, sa)
    res["engine_ms"] = timed_steps(estep, steps, flush)
    return res


def accum_case(api, kind, n, rho, steps, warmup, flush, exec_):
    import torch
    g = api.make_grid(api.map_kind[kind], 2, n, rho)
    side = g.cell_side()
    cells = api.tri_cells(side)
    a = torch.zeros(cells, dtype=torch.int32, device="cuda")

    def step(i):
        api.accum_device(g, a, 1, exec_)

    timed_steps(step, warmup, flush)
    ms = timed_steps(step, steps, flush)
    ok = bool((a == steps + warmup).all().item())
    return {"grid": f"{kind}({n}) rho={rho}", "side": side, "cells": cells, "ms": ms, "ok": ok, "step": step,
            "tensor": a}


def gcells(cells, ms):
    return cells / (ms * 1e-3) / 1e9


def energy_per_cell(sampler, step, cells, seconds=0.5):
    import torch
    e0 = sampler.energy_mj()
    if e0 is None:
        return None
    t0 = time.perf_counter()
    i = 0
    torch.cuda.synchronize()
    while time.perf_counter() - t0 < seconds:
        for _ in range(20):
            step(i)
            i += 1
        torch.cuda.synchronize()
    e1 = sampler.energy_mj()
    return (e1 - e0) * 1e-3 / (cells * i) if e1 is not None else None


def ncu_step_traffic():
    """DRAM bytes per C2 step (sum over the step's kernels) from the committed
    ncu summary (profiles/ncu_summary.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get("c2_step", {}).get("dram_bytes_per_step")
    except Exception:
        return None


def run_ours(args):
    import torch
    from paper_2208_11617_b200 import api

    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        from paper_2208_11617_b200 import dist as D
        return D.bench_sharded(args, api)

    peak, peak_src = load_peaks()
    flush = Flusher()
    desc, kind, n, rho = WORKLOADS[args.workload]
    sampler = ClockSampler(local)
    with sampler:
        h = ca_case(api, kind, n, rho, args.steps, args.warmup, flush)
    bb = ca_case(api, "bb", n - 1, rho, args.steps, args.warmup, flush)
    hb = ca_case(api, kind, n, rho, args.steps, args.warmup, flush, api.EXEC_BLOCK)
    bbb = ca_case(api, "bb", n - 1, rho, args.steps, args.warmup, flush, api.EXEC_BLOCK)
    cells = h["cells"]
    ms_h, ms_bb = statistics.mean(h["ms"]), statistics.mean(bb["ms"])
    value = gcells(cells, ms_h)
    achieved = 2.0 * cells / (ms_h * 1e-3) / 1e9

    # e2e: the reference-facing C ABI (smx_ca, launch_ca's semantics) with host
    # pinned buffers: H2D + one step + D2H inside the timed region
    host = torch.empty(cells, dtype=torch.uint8, pin_memory=True)
    api.life_init_device(3, h["side"], SEED, h["bufs"][0])
    host.copy_(h["bufs"][0].cpu())
    hnp = host.numpy()
    import ctypes as C
    from paper_2208_11617_b200 import _lib
    L = _lib.lib()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def e2e_step(i):
        _lib.check(L.smx_ca(C.byref(h["g"].raw), hnp.ctypes.data, cells, 1, api.EXEC_AUTO, 0, None, None, None,
                            stream))

    timed_steps(e2e_step, args.warmup)
    e2e_ms = statistics.mean(timed_steps(e2e_step, args.steps))

    j_h = energy_per_cell(sampler, h["step"], cells)
    j_bb = energy_per_cell(sampler, bb["step"], cells)
    cpu = cpu_baseline_c2(kind, n, rho, h["side"])
    configs = {} if args.no_configs else extra_configs(api, flush, sampler, peak, args)
    st = h["stage_ms"]
    line = {
        "metric": "Gcells/s (3-simplex CA step, H map) — BASELINE metric: Gcells/s and H-vs-BB speedup; "
                  "HBM GB/s vs peak; J/cell",
        "value": round(value, 3),
        "unit": "Gcells/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_h, 6),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (make_life_state seed 42, ~25% alive)",
        "impl": "ours",
        "config": {"workload": desc, "map": "h3d", "n_b": n, "rho": rho, "side": h["side"], "cells": cells,
                   "exec": "x-run (pack -> bit-sliced step -> unpack)",
                   "l2": "flushed before every timed step (256 MiB write)", "parallelism": "single GPU"},
        "h_vs_bb": round(ms_bb / ms_h, 3),
        "bb": {"grid": bb["grid"], "gcells_s": round(gcells(cells, ms_bb), 3), "ms_per_step": round(ms_bb, 6)},
        "block_scheme": {"h_gcells_s": round(gcells(cells, statistics.mean(hb["ms"])), 3),
                         "bb_gcells_s": round(gcells(cells, statistics.mean(bbb["ms"])), 3),
                         "h_vs_bb": round(statistics.mean(bbb["ms"]) / statistics.mean(hb["ms"]), 3),
                         "note": "the paper's launch model: one CTA per map block, rho^3 threads"},
        "engine": {"gcells_s": round(gcells(cells, statistics.mean(h["engine_ms"])), 3),
                   "ms_per_step": round(statistics.mean(h["engine_ms"]), 6),
                   "note": "multi-step launch_ca: bit shadow carried across steps (step + unpack per step)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": ncu_step_traffic(),
                     "kernel": "one u8->u8 CA step = k_pack_bits + k_ca_bits + k_unpack_bits",
                     "basis": "2 B per useful cell per step (u8 read + u8 write); per-launch CUDA events",
                     "stage_ms": {k: round(v, 6) for k, v in st.items()},
                     "peak_source": peak_src},
        "e2e": {"value": round(gcells(cells, e2e_ms), 3), "unit": "Gcells/s", "h2d_bytes_per_step": cells,
                "d2h_bytes_per_step": cells, "ms_per_step": round(e2e_ms, 4),
                "path": "smx_ca(host buffer, steps=1) through the C ABI"},
        "energy": {"j_per_cell_h": j_h, "j_per_cell_bb": j_bb},
        "cpu_baseline": cpu,
        "gpu_launches": 3 * args.steps,
        "clocks": sampler.summary(),
        "configs": configs,
    }
    return line


def cpu_baseline_c2(kind, n, rho, side):
    try:
        from oracle.oracle import H3D, Reference, reference_available
        if not reference_available():
            raise RuntimeError("oracle/_ref not built")
        R = Reference()
        s = R.make_life_state(3, side, SEED)
        _, _, _, secs = R.launch_ca(H3D, 3, n, rho, 1, s)
        cells = s.size
        return {"value": round(cells / secs / 1e9, 6), "unit": "Gcells/s", "cores": 1, "kind": "reference",
                "sample": f"reference launch_ca over grid_h3d({n}) rho={rho} (side {side}), 1 step, "
                          f"{secs:.2f} s, g++ -O3 -DNDEBUG (CMake Release flags)"}
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "Gcells/s", "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}


def extra_configs(api, flush, sampler, peak, args):
    """The other BASELINE configs at 1 GPU (H and BB, both execution schemes)."""
    import torch
    out = {}
    K, W = max(5, min(args.steps, 10)), 3

    def accum_pair(n, rho):
        r = {}
        for ex_name, ex in (("runs", api.EXEC_RUNS), ("block", api.EXEC_BLOCK)):
            h = accum_case(api, "h2d", n, rho, K, W, flush, ex)
            hms = statistics.mean(h["ms"])
            if ex_name == "runs":
                r["j_per_cell_h"] = energy_per_cell(sampler, h["step"], h["cells"], 0.3)
            del h["tensor"]
            torch.cuda.empty_cache()
            b = accum_case(api, "bb", n - 1, rho, K, W, flush, ex)
            bms = statistics.mean(b["ms"])
            if ex_name == "runs":
                r["j_per_cell_bb"] = energy_per_cell(sampler, b["step"], b["cells"], 0.3)
            gbs = 8.0 * h["cells"] / (hms * 1e-3) / 1e9
            r[ex_name] = {"h_gcells_s": round(gcells(h["cells"], hms), 2),
                          "bb_gcells_s": round(gcells(b["cells"], bms), 2),
                          "h_vs_bb": round(bms / hms, 3), "h_gb_s": round(gbs, 1),
                          "h_roofline_frac": round(gbs / peak, 4), "parity_ok": h["ok"] and b["ok"]}
            del b["tensor"]
            torch.cuda.empty_cache()
        r["cells"] = api.tri_cells((n - 1) * rho)
        r["grid"] = f"h2d({n}) vs bb({n - 1}), rho={rho}"
        return r

    def map_pair(m, n):
        gh = api.grid_h2d(n) if m == 2 else api.grid_h3d(n)
        gb = api.grid_bb(n - 1, m)
        res = {}
        for name, g in (("h", gh), ("bb", gb)):
            ms = timed_steps(lambda i: api.map_kernel_device(g), K + W)[W:]
            res[name + "_ms"] = round(statistics.mean(ms), 4)
            res[name + "_gblocks_s"] = round(g.blocks() / (statistics.mean(ms) * 1e-3) / 1e9, 2)
        res["h_vs_bb"] = round(res["bb_ms"] / res["h_ms"], 3)
        res["grid"] = f"MAP kernel h(n={n}) vs bb({n - 1}), rho=1, m={m} (same cell domain)"
        return res

    def ca_pair(n, rho):
        r = {}
        for ex_name, ex in (("runs", api.EXEC_RUNS), ("block", api.EXEC_BLOCK)):
            h = ca_case(api, "h3d", n, rho, K, W, flush, ex)
            if ex_name == "runs":
                r["j_per_cell_h"] = energy_per_cell(sampler, h["step"], h["cells"], 0.3)
            hms = statistics.mean(h["ms"])
            extra = {}
            if ex_name == "runs":
                extra = {"stage_ms": {k: round(v, 4) for k, v in h["stage_ms"].items()},
                         "engine_gcells_s": round(gcells(h["cells"], statistics.mean(h["engine_ms"])), 2)}
            del h
            torch.cuda.empty_cache()
            b = ca_case(api, "bb", n - 1, rho, K, W, flush, ex)
            if ex_name == "runs":
                r["j_per_cell_bb"] = energy_per_cell(sampler, b["step"], b["cells"], 0.3)
            bms = statistics.mean(b["ms"])
            cells = b["cells"]
            gbs = 2.0 * cells / (hms * 1e-3) / 1e9
            r[ex_name] = {"h_gcells_s": round(gcells(cells, hms), 2), "bb_gcells_s": round(gcells(cells, bms), 2),
                          "h_vs_bb": round(bms / hms, 3), "h_gb_s": round(gbs, 1),
                          "h_roofline_frac": round(gbs / peak, 4), **extra}
            del b
            torch.cuda.empty_cache()
        r["cells"] = api.tet_cells((n - 1) * rho)
        r["grid"] = f"h3d({n}) vs bb({n - 1}), rho={rho}"
        return r

    out["C1_accum_n1024"] = accum_pair(1024, 16)
    out["C1_map_kernel_2d"] = map_pair(2, 1024)
    out["C3_accum_n65536"] = accum_pair(4096, 16)
    out["C4_ca_n1024_1gpu"] = ca_pair(128, 8)
    out["C5_ca_n2048_1gpu"] = ca_pair(256, 8)
    out["map_kernel_3d"] = map_pair(3, 256)
    return out


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref) on the C2 workload:
    one launch_ca step per replica, one replica per host core (the reference is
    single-threaded within a launch, report.hpp:125-156)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return None
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import H3D, Reference, ncpu, reference_available
    desc, kind, n, rho = WORKLOADS[args.workload]
    side = (n - 1) * rho
    if not reference_available():
        return {"impl": "reference", "unavailable": "oracle/_ref (reference headers compiled) not built"}
    R = Reference()
    cores = ncpu()
    init = R.make_life_state(3, side, SEED)
    K = max(1, min(args.steps, 3))
    W = min(args.warmup, 1)

    def one(_):
        s = init.copy()
        _, _, _, secs = R.launch_ca(H3D, 3, n, rho, 1, s)
        return secs

    times = []
    with ThreadPoolExecutor(cores) as ex:
        for it in range(W + K):
            t0 = time.perf_counter()
            list(ex.map(one, range(cores)))
            dt = time.perf_counter() - t0
            if it >= W:
                times.append(dt)
    ms = statistics.mean(times) * 1e3
    cells = init.size
    value = cores * cells / (ms * 1e-3) / 1e9
    return {
        "metric": "Gcells/s (3-simplex CA step, H map) — BASELINE metric: Gcells/s and H-vs-BB speedup; "
                  "HBM GB/s vs peak; J/cell",
        "value": round(value, 6), "unit": "Gcells/s", "n_gpus": 0, "steps": K, "warmup": W,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic (make_life_state seed 42)", "impl": "reference",
        "config": {"workload": desc, "map": "h3d", "n_b": n, "rho": rho, "side": side, "cells": cells,
                   "parallelism": f"{cores} independent replicas, one per host core"},
        "cpu_baseline": {"value": round(value, 6), "unit": "Gcells/s", "cores": cores, "kind": "reference",
                         "sample": f"reference launch_ca(grid_h3d({n}), rho={rho}) 1 step x {cores} replicas "
                                   f"per bench step; K capped at 3 for a few-minute run"},
        "e2e": {"value": round(value, 6), "unit": "Gcells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config table")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None and env_int("RANK", 0) == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
