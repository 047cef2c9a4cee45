"""Benchmark driver (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-configs]

Headline workload (BASELINE.json configs[2], "C3", SURVEY 8(d) — the largest
single-GPU config): launch_accum over the 2-simplex n = 65536 through the H2D
block-space map, grid_h2d(4096), rho = 16: cell side 65520, 2,146,467,960 u32
cells (8.59 GB), zeros -> passes. A bench "step" is ONE launch_accum pass
(smx_accum on device buffers, EXEC_AUTO = the x-run kernel k_accum_runs, one
launch per pass); `value` = useful cells / device time (Gcells/s). The state
is 68x the 126 MB L2, so no flush is needed between steps (inputs larger than
L2). After the timed steps every cell must equal W + K (the reference's
launch_accum semantics, simulator.hpp:313-327), checked on the device.
BB (grid_bb(4095, 2), same cell domain) is timed the same way -> h_vs_bb.

`e2e` is the same pass through the reference-facing C ABI with HOST buffers
(smx_accum, device_ptr = 0, pinned host state): H2D 8.59 GB + pass + D2H
8.59 GB inside the timed region, every step.

`roofline` is for k_accum_runs (the step's only kernel), CUDA events on the
launching stream, SURVEY 8(d)'s basis of 8 B per useful cell (u32 read +
write); `traffic` is ncu's dram read + write per launch (profiles/).

`cpu_baseline` and `--impl reference` time the REFERENCE's own launch_accum
sweep (oracle/_ref: the unmodified headers compiled with the reference's
Release flags) over a bounded sample of the same grid — its first block rows —
one replica per host core (the reference is single-threaded per launch).

Also reported (`configs`): C1 ACCUM and the MAP kernel, C2/C4/C5 3-D Life
through the launch_ca engine (each final state hashed against the oracle's
golden, tests/golden/ca_full.json), single u8 steps, the rho sweep, the
paper's one-CTA-per-block launch model, the SURVEY 8(f) rows, and J/cell from
NVML (>= 5 s windows, idle power subtracted, 3 repeats).

Multi-GPU (`--gpus N`, N > 1; self-launches N ranks through torch.distributed.run
when not already under it): the C4 CA sharded over whole H levels
(paper_2208_11617_b200/dist.py) with the bit-tile halo exchange over NCCL.
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
METRIC = ("Gcells/s (2-simplex ACCUM through the H map, C3) — BASELINE metric: Gcells/s and H-vs-BB speedup; "
          "HBM GB/s vs peak; J/cell")
# the headline (BASELINE configs[2]): kind, n_b, rho of the H grid; BB uses n_b - 1
C3 = ("2-simplex n=65536 half-triangular accumulate (C3): launch_accum over grid_h2d(4096) rho=16, side 65520, "
      "2,146,467,960 u32 cells (8.59 GB), one pass per step", "h2d", 4096, 16)
C3_REF_HASH_1PASS = 18207742408615288078  # the reference's launch_accum, one pass
# the CA configs (engine calls of `steps` CA steps), golden keys in tests/golden/ca_full.json
CA_CONFIGS = {
    "C2_ca_n256": ("3-simplex n=256 CA (C2): launch_ca over grid_h3d(64) rho=4, side 252", 64, 4, 100,
                   "c2_rho4_100"),
    "C4_ca_n1024_1gpu": ("3-simplex n=1024 CA (C4) at 1 GPU: grid_h3d(128) rho=8, side 1016", 128, 8, 100,
                         "c4_rho8_100"),
    "C5_ca_n2048_1gpu": ("3-simplex n=2048 CA (C5) at 1 GPU: grid_h3d(256) rho=8, side 2040", 256, 8, 20,
                         "c5_rho8_20"),
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


def load_golden():
    p = os.path.join(ROOT, "tests", "golden", "ca_full.json")
    try:
        return json.load(open(p))["cases"]
    except Exception:
        return {}


def ncu_kernel_traffic(key: str):
    """dram read + write bytes per launch of a kernel from the committed ncu
    summary (profiles/ncu_summary.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        v = json.load(open(p)).get(key, {}).get("dram_bytes_per_launch")
        return float(v) if v is not None else None
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle-reason sampling through NVML."""

    def __init__(self, index=0, period=0.002):
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
        self._stop.clear()
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
    flush (when given) runs between timed steps, outside the events. Returns
    the ms list."""
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


def gcells(cells, ms):
    return cells / (ms * 1e-3) / 1e9


def device_hash(api, m, side, t) -> int:
    """simplex_grid_state::hash of a device state (copied to the host)."""
    return api.state_hash(m, side, t.cpu().numpy())


def energy_per_unit(sampler, step, units_per_step, seconds=5.0, repeats=3, idle_s=1.0):
    """J per unit from the NVML total-energy counter: `repeats` windows of at
    least `seconds` of back-to-back steps, each preceded by an idle window of
    `idle_s` whose average power is subtracted (net = gross - P_idle x t).
    Returns mean / min / max over the repeats, gross and net."""
    import torch
    if sampler.energy_mj() is None:
        return None
    rows = []
    i = 0
    for _ in range(repeats):
        torch.cuda.synchronize()
        time.sleep(0.2)
        e0, t0 = sampler.energy_mj(), time.perf_counter()
        time.sleep(idle_s)
        e1, t1 = sampler.energy_mj(), time.perf_counter()
        p_idle = (e1 - e0) * 1e-3 / (t1 - t0)
        n = 0
        e2, t2 = sampler.energy_mj(), time.perf_counter()
        while True:
            for _ in range(4):
                step(i)
                i += 1
                n += 1
            torch.cuda.synchronize()
            if time.perf_counter() - t2 >= seconds:
                break
        e3, t3 = sampler.energy_mj(), time.perf_counter()
        gross = (e3 - e2) * 1e-3
        rows.append({"gross": gross / (units_per_step * n), "net": (gross - p_idle * (t3 - t2)) / (units_per_step * n),
                     "idle_w": p_idle, "active_w": gross / (t3 - t2), "window_s": t3 - t2, "steps": n})

    def agg(k):
        v = [r[k] for r in rows]
        return {"mean": statistics.mean(v), "min": min(v), "max": max(v)}

    return {"j_per_unit_net": agg("net"), "j_per_unit_gross": agg("gross"), "idle_w": agg("idle_w"),
            "active_w": agg("active_w"), "window_s": round(min(r["window_s"] for r in rows), 2),
            "repeats": repeats}


# ---------------------------------------------------------------------------
# ACCUM (the headline)

def accum_case(api, kind, n, rho, steps, warmup, exec_, cells_t=None, flush=None):
    """`steps` timed launch_accum passes (device buffers) after `warmup`; the
    state is checked afterwards: every cell == warmup + steps."""
    import torch
    g = api.make_grid(api.map_kind[kind], 2, n, rho)
    side = g.cell_side()
    cells = api.tri_cells(side)
    a = cells_t if cells_t is not None else torch.empty(cells, dtype=torch.int32, device="cuda")
    a.zero_()

    def step(i):
        api.accum_device(g, a, 1, exec_)

    timed_steps(step, warmup, flush)
    ms = timed_steps(step, steps, flush)
    ok = bool((a == steps + warmup).all().item())
    return {"grid": f"{kind}({n}) rho={rho}", "side": side, "cells": cells, "ms": ms, "ok": ok, "step": step,
            "tensor": a, "g": g}


def run_ours(args):
    import torch
    from paper_2208_11617_b200 import api

    world = env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if world > 1:
        from paper_2208_11617_b200 import dist as D
        return D.bench_sharded(args, api)  # picks the device per backend
    torch.cuda.set_device(local)

    peak, peak_src = load_peaks()
    desc, kind, n, rho = C3
    sampler = ClockSampler(local)
    side = (n - 1) * rho
    cells = api.tri_cells(side)
    buf = torch.empty(cells, dtype=torch.int32, device="cuda")
    with sampler:
        h = accum_case(api, kind, n, rho, args.steps, args.warmup, api.EXEC_AUTO, buf)
    clocks = sampler.summary()
    ms_h = statistics.mean(h["ms"])
    h_ok = h["ok"]
    value = gcells(cells, ms_h)
    # the same state after exactly ONE pass must hash to the reference's
    # Appendix A value (state hash over all 8.59 GB on the host)
    buf.zero_()
    api.accum_device(h["g"], buf, 1, api.EXEC_AUTO)
    one_pass_hash = device_hash(api, 2, side, buf)
    bb = accum_case(api, "bb", n - 1, rho, args.steps, args.warmup, api.EXEC_AUTO, buf)
    ms_bb = statistics.mean(bb["ms"])
    # the paper's one-CTA-per-block launch model (same state, same check)
    Kb = max(3, min(args.steps, 10))
    hb = accum_case(api, kind, n, rho, Kb, 3, api.EXEC_BLOCK, buf)
    bbb = accum_case(api, "bb", n - 1, rho, Kb, 3, api.EXEC_BLOCK, buf)
    ms_hb, ms_bbb = statistics.mean(hb["ms"]), statistics.mean(bbb["ms"])
    block_model = {"note": "the paper's launch model: one CTA per map block, rho^2 = 256 threads (EXEC_BLOCK)",
                   "h_gcells_s": round(gcells(cells, ms_hb), 3), "bb_gcells_s": round(gcells(cells, ms_bbb), 3),
                   "h_vs_bb": round(ms_bbb / ms_hb, 3), "parity_ok": hb["ok"] and bbb["ok"],
                   "h_roofline_frac": round(8.0 * cells / (ms_hb * 1e-3) / 1e9 / peak, 4)}

    # roofline: the step is ONE k_accum_runs launch (events on its stream)
    achieved = 8.0 * cells / (ms_h * 1e-3) / 1e9
    traffic = ncu_kernel_traffic("c3_accum_runs")

    # e2e: the reference-facing C ABI (smx_accum = launch_accum) with a pinned
    # host state: H2D + pass + D2H inside the timed region
    del hb, bbb
    host = torch.zeros(cells, dtype=torch.int32, pin_memory=True)
    hnp = host.numpy()
    import ctypes as C
    from paper_2208_11617_b200 import _lib
    L = _lib.lib()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def e2e_call(i):
        _lib.check(L.smx_accum(C.byref(h["g"].raw), hnp.ctypes.data, cells, 1, api.EXEC_AUTO, 0, None, None,
                               stream))

    timed_steps(e2e_call, args.warmup)
    e2e_ms_list = timed_steps(e2e_call, args.steps)
    e2e_ms = statistics.mean(e2e_ms_list)
    e2e_ok = bool((host == args.steps + args.warmup).all().item())
    h2d_ms = statistics.median(timed_steps(lambda i: buf.copy_(host, non_blocking=True), 3))
    d2h_ms = statistics.median(timed_steps(lambda i: host.copy_(buf, non_blocking=True), 3))
    # both directions at once (two streams, halves of the state each way): the
    # PCIe duplex floor the pipelined host path runs against
    half = cells // 2
    up, down = torch.cuda.Stream(), torch.cuda.Stream()

    def duplex(i):
        cur = torch.cuda.current_stream()
        up.wait_stream(cur)
        down.wait_stream(cur)
        with torch.cuda.stream(up):
            buf[:half].copy_(host[:half], non_blocking=True)
        with torch.cuda.stream(down):
            host[half:].copy_(buf[half:], non_blocking=True)
        cur.wait_stream(up)
        cur.wait_stream(down)

    duplex_ms = statistics.median(timed_steps(duplex, 3))
    del host, hnp
    api.release_scratch()  # the 8.59 GB staging pool of the host-buffer call

    energy = {}
    if not args.no_energy:
        energy["C3_h"] = energy_per_unit(sampler, h["step"], cells)
        energy["C3_bb"] = energy_per_unit(sampler, bb["step"], cells)
    del h["tensor"], bb["tensor"]
    del buf
    torch.cuda.empty_cache()
    cpu = cpu_baseline_c3(kind, n, rho)
    configs = {} if args.no_configs else extra_configs(api, sampler, peak, args, energy)
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "Gcells/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_h, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (zero state; every pass increments every cell once)",
        "impl": "ours",
        "config": {"workload": desc, "map": "h2d", "n_b": n, "rho": rho, "side": side, "cells": cells,
                   "passes_per_step": 1, "exec": "x-run (k_accum_runs: 32 blocks mapped lane-parallel per CTA, "
                                                 "tiles merged into runs, 16-byte vectors)",
                   "l2": "no flush: the 8.59 GB state is 68x the L2 (inputs larger than L2)",
                   "parallelism": "single GPU"},
        "parity": {"all_cells_equal_passes": h_ok and bb["ok"], "bb_ok": bb["ok"], "e2e_ok": e2e_ok,
                   "one_pass_state_hash": str(one_pass_hash),
                   "one_pass_hash_equals_reference": one_pass_hash == C3_REF_HASH_1PASS,
                   "reference_hash": str(C3_REF_HASH_1PASS)},
        "h_vs_bb": round(ms_bb / ms_h, 3),
        "bb": {"grid": bb["grid"], "gcells_s": round(gcells(cells, ms_bb), 3), "ms_per_step": round(ms_bb, 5)},
        "block_model": block_model,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "frac_vs_nominal_8tbs": round(achieved / 8000.0, 4),
                     "kernel": "k_accum_runs<H2D> (the step's only launch)",
                     "kernel_ms": round(ms_h, 6), "launches_per_step": 1,
                     "basis": "8 B per useful cell (u32 read + u32 write, SURVEY 8(d)) x 2,146,467,960 cells per "
                              "launch / mean launch time (CUDA events on the launching stream)",
                     "peak_source": peak_src},
        "e2e": {"value": round(gcells(cells, e2e_ms), 3), "unit": "Gcells/s",
                "h2d_bytes_per_step": 4 * cells, "d2h_bytes_per_step": 4 * cells, "ms_per_step": round(e2e_ms, 3),
                "path": "smx_accum(pinned host state, passes=1, EXEC_AUTO) through the C ABI",
                "h2d_ms": round(h2d_ms, 3), "d2h_ms": round(d2h_ms, 3),
                "pcie_gb_s": round(8.0 * cells / ((h2d_ms + d2h_ms) * 1e-3) / 1e9, 1),
                "duplex_half_each_way_ms": round(duplex_ms, 3),
                "duplex_gb_s": round(4.0 * cells / (duplex_ms * 1e-3) / 1e9, 1),
                "note": "H2D and D2H of the whole state overlap chunk by chunk (smx_accum's pipelined host path); "
                        "duplex_gb_s is both directions moving at once (half the state each way)"},
        "energy": energy,
        "cpu_baseline": cpu,
        "gpu_launches": args.steps,
        "clocks": clocks,
        "configs": configs,
    }
    return line


def ref_sample_rows_threads():
    """Reference-sample sizing: block rows of grid_h2d(4096) rho=16 per replica
    (each row is 524,288 cells, ~3 ms on one core) and the replica count (one
    per host core, bounded by ~0.8 GB touched per replica vs available RAM)."""
    from oracle.oracle import ncpu
    cores = ncpu()
    try:
        avail_gb = int(open("/proc/meminfo").read().split("MemAvailable:")[1].split()[0]) / 1e6
    except Exception:
        avail_gb = 16.0
    return 256, max(1, min(cores, int(0.5 * avail_gb / 0.8))), cores


def cpu_baseline_c3(kind, n, rho):
    """The reference's own launch_accum sweep (oracle/_ref) on the host cores:
    a bounded sample of C3 (its first 256 block rows = 134 M cells per
    replica), one replica per core, 1 warm + 3 timed repetitions."""
    try:
        from oracle.oracle import H2D, Reference, reference_available
        if not reference_available():
            raise RuntimeError("oracle/_ref not built")
        rows, threads, cores = ref_sample_rows_threads()
        secs, useful = Reference().accum_sample(H2D, 2, n, rho, rows, threads, 1, 3)
        s = statistics.median(secs)
        return {"value": round(threads * useful / s / 1e9, 4), "unit": "Gcells/s", "cores": threads,
                "kind": "reference",
                "sample": f"reference launch_accum sweep (accounted_sweep + ++cells[idx], simulator.hpp:277-327) "
                          f"over the first {rows} block rows of grid_h2d({n}) rho={rho} ({useful} cells of the "
                          f"C3 state) x {threads} concurrent replicas (host has {cores} cores), median of 3 "
                          f"({s:.2f} s each); g++ -O3 -DNDEBUG (the reference's Release flags)"}
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "Gcells/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}


# ---------------------------------------------------------------------------
# the other BASELINE configs at 1 GPU

def make_state(api, kind, n, rho):
    import torch
    g = api.make_grid(api.map_kind[kind], 3, n, rho)
    side = g.cell_side()
    cells = api.tet_cells(side)
    a = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
    b = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
    api.life_init_device(3, side, SEED, a)
    return g, side, cells, a, b


def engine_case(api, kind, n, rho, ca_steps, iters, warmup, flush, golden_key=None, golden=None):
    """`iters` launch_ca calls of `ca_steps` CA steps each (device buffers, AUTO
    = bit-shadow engine), L2 flushed before each call; ms per call. Then the
    state is re-seeded, ONE call is made and its final state hashed against
    the oracle's golden for (side, ca_steps)."""
    g, side, cells, a, b = make_state(api, kind, n, rho)

    def call(i):
        api.ca_device(g, a, ca_steps, api.EXEC_AUTO, b)

    timed_steps(call, warmup, flush)
    ms = timed_steps(call, iters, flush)
    check = None
    if golden_key and golden and golden_key in golden:
        want = golden[golden_key]
        assert want["side"] == side and want["steps"] == ca_steps, golden_key
        api.life_init_device(3, side, SEED, a)
        call(0)
        got = device_hash(api, 3, side, a)
        check = {"golden": golden_key, "hash": str(got), "ok": str(got) == str(want["final_hash"])}
    return {"grid": f"{kind}({n}) rho={rho}", "side": side, "cells": cells, "g": g, "ms": ms, "call": call,
            "bufs": (a, b), "check": check}


def engine_kernel_ms(api, g, a, ca_steps, iters):
    """Average duration of the engine stage (smx_bits_run: the plan kernel plus
    ONE persistent k_ca_bits_run launch of `ca_steps` steps), events on the
    launching stream around each call; returns ms per call."""
    import torch
    sa, sb = api.bits_buffer(g), api.bits_buffer(g)
    api.bits_pack_device(g, a, sa)
    api.bits_run_device(g, sa, sb, ca_steps)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for e0, e1 in ev:
        e0.record()
        api.bits_run_device(g, sa, sb, ca_steps)
        e1.record()
    torch.cuda.synchronize()
    return statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev)


def step_case(api, kind, n, rho, iters, warmup, flush, exec_):
    """Single u8 -> u8 CA steps (smx_ca_step), L2 flushed before each. ms per step."""
    g, side, cells, a, b = make_state(api, kind, n, rho)
    bufs = [a, b]

    def step(i):
        api.ca_step_device(g, bufs[i % 2], bufs[(i + 1) % 2], exec_)

    timed_steps(step, warmup, flush)
    return {"grid": f"{kind}({n}) rho={rho}", "cells": cells, "ms": timed_steps(step, iters, flush), "step": step}


def extra_configs(api, sampler, peak, args, energy):
    """The other BASELINE configs at 1 GPU (H and BB, both execution schemes)."""
    import torch
    out = {}
    flush = Flusher()
    K, W = max(5, min(args.steps, 10)), 3
    golden = load_golden()

    def accum_pair(n, rho):
        r = {}
        for ex_name, ex in (("runs", api.EXEC_RUNS), ("block", api.EXEC_BLOCK)):
            h = accum_case(api, "h2d", n, rho, K, W, ex, flush=flush)
            hms = statistics.mean(h["ms"])
            del h["tensor"]
            b = accum_case(api, "bb", n - 1, rho, K, W, ex, flush=flush)
            bms = statistics.mean(b["ms"])
            gbs = 8.0 * h["cells"] / (hms * 1e-3) / 1e9
            r[ex_name] = {"h_gcells_s": round(gcells(h["cells"], hms), 2),
                          "bb_gcells_s": round(gcells(b["cells"], bms), 2),
                          "h_vs_bb": round(bms / hms, 3), "h_gb_s": round(gbs, 1),
                          "h_roofline_frac": round(gbs / peak, 4), "parity_ok": h["ok"] and b["ok"]}
            del b["tensor"]
            torch.cuda.empty_cache()
        r["cells"] = api.tri_cells((n - 1) * rho)
        r["grid"] = f"h2d({n}) vs bb({n - 1}), rho={rho}; L2 flushed before every pass"
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

    def ca_pair(label, n, rho, ca_steps, key, with_energy):
        """CA at 1 GPU: launch_ca engine calls of `ca_steps` steps (H and BB,
        each final state hashed against the oracle golden), the dominant
        kernel's roofline, and single u8 -> u8 steps."""
        r = {"grid": f"h3d({n}) vs bb({n - 1}), rho={rho}", "ca_steps_per_call": ca_steps,
             "l2": "flushed before every call",
             "engine_kind": api.ca_engine(api.make_grid(api.map_kind.h3d, 3, n, rho))}
        h = engine_case(api, "h3d", n, rho, ca_steps, K if ca_steps * n <= 12800 else 3, 1, flush, key, golden)
        cells = h["cells"]
        r["cells"] = cells
        r["side"] = h["side"]
        hms = statistics.mean(h["ms"])
        kms = engine_kernel_ms(api, h["g"], h["bufs"][0], ca_steps, 3) / ca_steps
        if with_energy and not args.no_energy:
            energy[label + "_h"] = energy_per_unit(sampler, h["call"], cells * ca_steps)
        r["parity_h"] = h["check"]
        del h
        torch.cuda.empty_cache()
        b = engine_case(api, "bb", n - 1, rho, ca_steps, K if ca_steps * n <= 12800 else 3, 1, flush, key, golden)
        bms = statistics.mean(b["ms"])
        if with_energy and not args.no_energy:
            energy[label + "_bb"] = energy_per_unit(sampler, b["call"], cells * ca_steps)
        r["parity_bb"] = b["check"]
        del b
        torch.cuda.empty_cache()
        gbs = 2.0 * cells * ca_steps / (hms * 1e-3) / 1e9
        kgbs = 2.0 * cells / (kms * 1e-3) / 1e9
        r["engine"] = {"h_gcell_steps_s": round(gcells(cells * ca_steps, hms), 2),
                       "bb_gcell_steps_s": round(gcells(cells * ca_steps, bms), 2),
                       "h_vs_bb": round(bms / hms, 3), "h_ms_per_call": round(hms, 4),
                       "h_u8_basis_gb_s": round(gbs, 1), "h_roofline_frac": round(gbs / peak, 4),
                       "run_kernel_ms_per_step": round(kms, 5), "run_kernel_roofline_frac": round(kgbs / peak, 4),
                       # the bytes the bit engine must move (bit shadow read + written once per step)
                       # against HBM: it is instruction bound (ncu: ALU pipe / issue), not HBM bound
                       "run_kernel_bits_basis_frac": round(2.0 * cells / 8 / (kms * 1e-3) / 1e9 / peak, 4),
                       "run_kernel_bound": "instruction issue (LOP3 on the ALU pipe + shared-memory latency; "
                                           "DESIGN.md section 6)",
                       "note": "pack + plan + ONE persistent launch of ca_steps steps + unpack per call; "
                               "2 B/cell/step u8 basis"}
        for name, ex in (("single_auto", api.EXEC_AUTO), ("single_fused", api.EXEC_RUNS),
                         ("single_block", api.EXEC_BLOCK)):
            K1 = 3 if name == "single_block" else K
            sh = step_case(api, "h3d", n, rho, K1, 1, flush, ex)
            mh = statistics.mean(sh["ms"])
            del sh
            torch.cuda.empty_cache()
            sb = step_case(api, "bb", n - 1, rho, K1, 1, flush, ex)
            mb = statistics.mean(sb["ms"])
            del sb
            torch.cuda.empty_cache()
            g1 = 2.0 * cells / (mh * 1e-3) / 1e9
            r[name] = {"h_gcells_s": round(gcells(cells, mh), 2), "bb_gcells_s": round(gcells(cells, mb), 2),
                       "h_vs_bb": round(mb / mh, 3), "h_ms": round(mh, 4), "h_roofline_frac": round(g1 / peak, 4)}
        return r

    out["C1_accum_n1024"] = accum_pair(1024, 16)
    out["C1_map_kernel_2d"] = map_pair(2, 1024)
    # the C3 cell domain (side ~65.5 K, 8.6 GB) at smaller tiles: the map's
    # per-block share grows as rho falls, and H's half-size grid shows
    sweep = {}
    for n, rho in ((32768, 2), (16384, 4), (8192, 8), (4096, 16)):
        h = accum_case(api, "h2d", n, rho, K, W, api.EXEC_RUNS)
        hms = statistics.mean(h["ms"])
        del h["tensor"]
        torch.cuda.empty_cache()
        b = accum_case(api, "bb", n - 1, rho, K, W, api.EXEC_RUNS)
        bms = statistics.mean(b["ms"])
        del b["tensor"]
        torch.cuda.empty_cache()
        gbs = 8.0 * h["cells"] / (hms * 1e-3) / 1e9
        sweep[f"rho{rho}"] = {"grid": f"h2d({n}) vs bb({n - 1}), rho={rho}, side {h['side']}",
                              "h_gcells_s": round(gcells(h["cells"], hms), 2),
                              "bb_gcells_s": round(gcells(b["cells"], bms), 2), "h_vs_bb": round(bms / hms, 3),
                              "h_roofline_frac": round(gbs / peak, 4), "parity_ok": h["ok"] and b["ok"]}
    out["C3_accum_rho_sweep"] = sweep
    for label, (desc, n, rho, ca_steps, key) in CA_CONFIGS.items():
        out[label] = ca_pair(label, n, rho, ca_steps, key, label != "C2_ca_n256")
        out[label]["workload"] = desc
    # rho sweep at the same n = 2048 cell scale (trade map
    # amortisation against the BB/H block ratio); r/beta are fixed at (2, 2)
    # by the executable map
    from paper_2208_11617_b200 import analysis as A
    ranked = A.optimize_params(3, 8, 8, 256)
    out["C5_r_beta_sweep"] = {
        "note": "analytical (analysis.hpp restated, exact): optimize_params(m=3, 1/r<=8, beta<=8, n_eval=256); "
                "the executable H3D is the (2, 2) family — every other family under-covers (alpha < 0)",
        "top": [{"inv_r": p.inv_r, "beta": p.beta, "alpha": str(r.alpha), "n0": r.n0 if r.found else None}
                for p, r in ranked[:6]], "families": len(ranked)}
    c5r4 = engine_case(api, "h3d", 512, 4, 20, 3, 1, flush, "c5_rho4_20", golden)
    out["C5_rho4_engine"] = {"grid": "h3d(512) rho=4", "side": c5r4["side"], "cells": c5r4["cells"],
                             "h_gcell_steps_s": round(gcells(c5r4["cells"] * 20, statistics.mean(c5r4["ms"])), 2),
                             "parity": c5r4["check"]}
    del c5r4
    torch.cuda.empty_cache()
    c5r16 = engine_case(api, "h3d", 128, 16, 20, 3, 1, flush, "c5_rho16_20", golden)
    out["C5_rho16_engine"] = {"grid": "h3d(128) rho=16", "side": c5r16["side"], "cells": c5r16["cells"],
                              "h_gcell_steps_s": round(gcells(c5r16["cells"] * 20, statistics.mean(c5r16["ms"])), 2),
                              "parity": c5r16["check"], "engine_kind": "column"}
    del c5r16
    torch.cuda.empty_cache()
    out["map_kernel_3d"] = map_pair(3, 256)
    out.update(next_rows(api, flush, peak, K))
    out["cpu_reference"] = cpu_reference_rows()
    out["h_vs_bb_summary"] = h_vs_bb_summary(out)
    return out


def h_vs_bb_summary(configs):
    """The paper's headline comparison in one place: where the work is per
    launched block (the MAP kernel, the one-CTA-per-block launch model) H's
    fewer blocks show as the block ratio; the x-run schemes make BB's Void
    blocks nearly free, so the streaming kernels run at the same roof at
    rho = 16 — at smaller tiles (the C3 rho sweep) the per-block share grows
    and H's half-size grid keeps a lead."""
    out = {}
    pick = {"map_kernel_2d": ("C1_map_kernel_2d", None), "map_kernel_3d": ("map_kernel_3d", None),
            "accum_xrun_c1": ("C1_accum_n1024", "runs"), "accum_block_model_c1": ("C1_accum_n1024", "block"),
            "accum_xrun_c3_rho8": ("C3_accum_rho_sweep", "rho8"), "accum_xrun_c3_rho4": ("C3_accum_rho_sweep", "rho4"),
            "accum_xrun_c3_rho2": ("C3_accum_rho_sweep", "rho2"),
            "ca_engine_c2": ("C2_ca_n256", "engine"), "ca_engine_c4": ("C4_ca_n1024_1gpu", "engine"),
            "ca_engine_c5": ("C5_ca_n2048_1gpu", "engine"),
            "ca_single_step_c5": ("C5_ca_n2048_1gpu", "single_auto"),
            "ca_block_model_c5_1step": ("C5_ca_n2048_1gpu", "single_block")}
    for k, (cfg, sub) in pick.items():
        c = configs.get(cfg)
        if c is not None:
            c = c.get(sub) if sub else c
            out[k] = c.get("h_vs_bb") if isinstance(c, dict) else None
    return out


def cpu_reference_rows():
    """The reference's own launch_* (oracle/_ref, Release flags) on one host
    core, bounded samples beside the GPU configs (Gcells/s per call)."""
    try:
        from oracle.oracle import H2D, H3D, Reference, reference_available
        if not reference_available():
            return {"unavailable": "oracle/_ref not built"}
        R = Reference()
        out = {}
        _, cnt, _, secs = R.launch_accum(H2D, 2, 1024, 16, passes=1)
        out["accum_C1_h2d1024_rho16"] = {"gcells_s": round(cnt[3] / secs / 1e9, 4), "seconds": round(secs, 3)}
        t0 = time.perf_counter()
        _, cnt, _ = R.launch_edm(H2D, 1024, 4, 7)
        dt = time.perf_counter() - t0
        out["edm_h2d1024_rho4"] = {"gcells_s": round(cnt[3] / dt / 1e9, 4), "seconds": round(dt, 3),
                                   "note": "side 4092 sample (the GPU row is side 16368)"}
        s = R.make_life_state(2, 1023, SEED)
        _, cnt, _, secs = R.launch_ca(H2D, 2, 1024, 1, 1, s)
        out["ca2d_periodic_h2d1024_1step"] = {"gcells_s": round(cnt[3] / secs / 1e9, 4), "seconds": round(secs, 3),
                                              "note": "side 1023 sample"}
        s = R.make_life_state(3, 252, SEED)
        _, cnt, _, secs = R.launch_ca(H3D, 3, 64, 4, 1, s)
        out["ca3d_C2_1step"] = {"gcells_s": round(cnt[3] / secs / 1e9, 6), "seconds": round(secs, 3)}
        out["cores"] = 1
        return out
    except Exception as e:  # pragma: no cover
        return {"unavailable": str(e)}


def next_rows(api, flush, peak, K):
    """SURVEY 8(f) rows at 1 GPU: general-n H (trapezoid bands / padded) ACCUM
    at the C3 scale, EDM (f64, 8 B written per cell) and the periodic 2-D Life
    step through H2D vs BB, and the GPU cover-verification sweep."""
    import torch
    out = {}

    def timed(fn, iters):
        timed_steps(lambda i: fn(), 2, flush)
        return statistics.mean(timed_steps(lambda i: fn(), iters, flush))

    acc = {}
    for name, g in (("trapezoid_n4097_T4", api.make_grid(api.map_kind.h2d_trapezoid, 2, 4097, 16, 4)),
                    ("padded_n3000", api.make_grid(api.map_kind.h2d_padded, 2, 3000, 16)),
                    ("bb_n3000", api.make_grid(api.map_kind.bb, 2, 3000, 16))):
        cells = api.tri_cells(g.cell_side())
        a = torch.zeros(cells, dtype=torch.int32, device="cuda")
        ms = timed(lambda: api.accum_device(g, a, 1, api.EXEC_RUNS), K)
        acc[name] = {"side": g.cell_side(), "cells": cells, "gcells_s": round(gcells(cells, ms), 2),
                     "roofline_frac": round(8.0 * cells / (ms * 1e-3) / 1e9 / peak, 4)}
        del a
        torch.cuda.empty_cache()
    out["F1_general_n_accum"] = acc

    gh, gb = api.make_grid(api.map_kind.h2d, 2, 1024, 16), api.make_grid(api.map_kind.bb, 2, 1023, 16)
    side = gh.cell_side()
    cells = api.tri_cells(side)
    pts = torch.from_numpy(api.make_edm_points(side, 7)).cuda()
    e = torch.empty(cells, dtype=torch.float64, device="cuda")
    edm = {"side": side, "cells": cells}
    for ex_name, ex in (("runs", api.EXEC_RUNS), ("block", api.EXEC_BLOCK)):
        mh = timed(lambda: api.edm_device(gh, pts, e, ex), K)
        mb = timed(lambda: api.edm_device(gb, pts, e, ex), K)
        edm[ex_name] = {"h_gcells_s": round(gcells(cells, mh), 2), "bb_gcells_s": round(gcells(cells, mb), 2),
                        "h_vs_bb": round(mb / mh, 3),
                        "h_roofline_frac": round(8.0 * cells / (mh * 1e-3) / 1e9 / peak, 4)}
    del e
    torch.cuda.empty_cache()
    out["F2_edm_n1024"] = edm

    a = torch.empty(cells, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    api.life_init_device(2, side, SEED, a)
    ca = {"side": side, "cells": cells}
    for ex_name, ex in (("runs", api.EXEC_RUNS), ("block", api.EXEC_BLOCK)):
        mh = timed(lambda: api.ca_step_device(gh, a, b, ex), K)
        mb = timed(lambda: api.ca_step_device(gb, a, b, ex), K)
        ca[ex_name] = {"h_gcells_s": round(gcells(cells, mh), 2), "bb_gcells_s": round(gcells(cells, mb), 2),
                       "h_vs_bb": round(mb / mh, 3),
                       "h_roofline_frac": round(2.0 * cells / (mh * 1e-3) / 1e9 / peak, 4)}
    del a, b
    torch.cuda.empty_cache()
    out["F3_ca2d_periodic_n1024"] = ca

    from paper_2208_11617_b200 import report as rp
    t0 = time.perf_counter()
    rows = rp.verify_sweep(api.map_kind.h2d_trapezoid, 2, list(range(2, 4097)), 1, 4)
    out["F4_verify_sweep"] = {"sweep": "verify_sweep(trapezoid, m=2, n=2..4096, T=4) on the GPU",
                              "grids": len(rows), "all_exact": all(r.exact for r in rows),
                              "seconds": round(time.perf_counter() - t0, 2)}
    return out


def run_reference(args):
    """`--impl reference`: the reference's own CPU launch_accum (oracle/_ref)
    on the headline C3 grid, all host cores: each bench step is a bounded
    sample (the first 256 block rows of grid_h2d(4096) rho=16, 134 M cells)
    per replica, one replica per core; W untimed + K timed steps as asked.
    The value is Gcells/s, the same metric as ours. Rank 0 only."""
    if env_int("RANK", 0) != 0:
        return None
    from oracle.oracle import H2D, Reference, reference_available
    desc, kind, n, rho = C3
    side = (n - 1) * rho
    if not reference_available():
        return {"impl": "reference", "unavailable": "oracle/_ref (reference headers compiled) not built"}
    rows, threads, cores = ref_sample_rows_threads()
    K, W = max(1, args.steps), max(0, args.warmup)
    secs, useful = Reference().accum_sample(H2D, 2, n, rho, rows, threads, W, K)
    ms = statistics.mean(secs) * 1e3
    value = threads * useful / (ms * 1e-3) / 1e9
    sample = (f"reference launch_accum sweep (accounted_sweep + ++cells[idx], simulator.hpp:277-327) over the first "
              f"{rows} block rows of grid_h2d({n}) rho={rho} ({useful} of the {api_tri_cells(side)} C3 cells) per "
              f"replica, {threads} concurrent replicas (one per core; host has {cores})")
    return {
        "metric": METRIC,
        "value": round(value, 4), "unit": "Gcells/s", "n_gpus": 0, "steps": K, "warmup": W,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic (zero state)", "impl": "reference",
        "config": {"workload": desc, "map": "h2d", "n_b": n, "rho": rho, "side": side, "cells": api_tri_cells(side),
                   "parallelism": f"{threads} independent replicas, one per host core"},
        "cpu_baseline": {"value": round(value, 4), "unit": "Gcells/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "Gcells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def api_tri_cells(side):
    return side * (side + 1) // 2


def self_launch(args):
    """bench.py --gpus N outside torchrun: re-run this script as N ranks."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config table")
    ap.add_argument("--no-energy", action="store_true", help="skip the NVML energy windows")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world = env_int("WORLD_SIZE", 0)
    if args.impl == "ours":
        if args.gpus > 1 and world == 0:
            self_launch(args)
        if world and world != args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
            sys.exit(2)
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None and env_int("RANK", 0) == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
