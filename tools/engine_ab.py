"""A/B timing of the CA engines (run on the GPU box):

    SMX_CA_ENGINE=cols|chunks python tools/engine_ab.py [n rho steps kind ...]

Per case: launch_ca engine stage (smx_bits_run: plan + ONE persistent launch
of `steps` steps) timed with CUDA events, median of 5 after 2 warm-ups; the
state hash after one full launch_ca call is checked against the oracle golden
when one exists. Prints one JSON line per case."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2208_11617_b200 import api  # noqa: E402

CASES = [("h3d", 64, 4, 100), ("bb", 63, 4, 100), ("h3d", 128, 8, 100), ("bb", 127, 8, 100),
         ("h3d", 256, 8, 20), ("bb", 255, 8, 20), ("h3d", 512, 4, 20)]
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "ca_full.json")))["cases"]


def main():
    cases = CASES
    if len(sys.argv) > 1:
        a = sys.argv[1:]
        cases = [(a[i + 3], int(a[i]), int(a[i + 1]), int(a[i + 2])) for i in range(0, len(a), 4)]
    for kind, n, rho, steps in cases:
        g = api.make_grid(api.map_kind[kind], 3, n, rho)
        side = g.cell_side()
        cells = api.tet_cells(side)
        u8 = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
        api.life_init_device(3, side, 42, u8)
        A, B = api.bits_buffer(g), api.bits_buffer(g)
        api.bits_pack_device(g, u8, A)
        for _ in range(2):
            api.bits_run_device(g, A, B, steps)
        ms = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            api.bits_run_device(g, A, B, steps)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        m = statistics.median(ms)
        api.life_init_device(3, side, 42, u8)
        api.ca_device(g, u8, steps, api.EXEC_BITS)
        h = api.state_hash(3, side, u8.cpu().numpy())
        gold = next((v for v in GOLD.values() if v["side"] == side and v["steps"] == steps), None)
        print(json.dumps({"engine": os.environ.get("SMX_CA_ENGINE", "auto"), "grid": f"{kind}({n}) rho={rho}",
                          "side": side, "steps": steps, "ms_per_call": round(m, 4),
                          "us_per_step": round(1000 * m / steps, 2),
                          "gcell_steps_s": round(cells * steps / (m * 1e-3) / 1e9, 1),
                          "u8_roof_frac": round(2 * cells * steps / (m * 1e-3) / 6529.7e9, 3),
                          "hash_ok": None if gold is None else str(h) == str(gold["final_hash"])}), flush=True)
        del u8, A, B
        api.release_scratch()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
