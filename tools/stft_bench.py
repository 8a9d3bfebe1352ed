"""STFT throughput: StftPlan over a synthetic complex64
signal in HBM, frames of n points every hop samples, with and without a Hann
window; 16 n algorithmic bytes per frame (the frame read once, its spectrum
written once); CUDA events, best of 10 after warm-up; kernels per exec from the
plan info.
  python tools/stft_bench.py [--n 65536,16384,1024] [--gib 2] [--json OUT]"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", default="65536,16384,1024")
ap.add_argument("--gib", type=float, default=2.0)
ap.add_argument("--json", default=None)
a = ap.parse_args()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
rows = []
for n in [int(v) for v in a.n.split(",")]:
    frames = int(a.gib * 2 ** 30) // (8 * n)
    for hop in (n // 2, n // 2 + 1):
        sig = torch.randn((frames - 1) * hop + n, dtype=torch.complex64, device="cuda")
        out = torch.empty((frames, n), dtype=torch.complex64, device="cuda")
        for win in (False, True):
            w = [0.5 - 0.5 * math.cos(2 * math.pi * i / n) for i in range(n)] if win else None
            with bf.StftPlan(n, hop, frames, window=w) as p:
                for _ in range(3):
                    p.exec(sig, out)
                best = 1e9
                for _ in range(10):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record(); p.exec(sig, out); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
                kpe = p.info()["kernels_per_exec"]
            gbs = 16.0 * n * frames / (best * 1e-3) / 1e9
            row = {"n": n, "hop": hop, "window": win, "frames": frames, "ms": best, "alg_GBps": gbs, "frac": gbs / peak,
                   "kernels": kpe}
            rows.append(row)
            print(f"stft n={n:<6} hop={hop:<6} window={int(win)} frames={frames:<6} {best:7.3f} ms {gbs:7.1f} GB/s "
                  f"{gbs/peak:6.1%} kernels={kpe}", flush=True)
        del sig, out
if a.json:
    json.dump(rows, open(a.json, "w"), indent=1)
