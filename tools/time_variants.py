"""Time every kernel variant over a range of N with CUDA events (in-HBM,
out-of-place, >= 1 GiB per direction so inputs exceed L2).  Prints one line
per (N, variant, cluster size) with ms/exec, algorithmic GB/s (16 N bytes per
record) and the fraction of the measured HBM copy bandwidth.

  python tools/time_variants.py [--min 8] [--max 22] [--bytes 2GiB] [--variants 1,2,3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402
from synth import gpu as sg  # noqa: E402


def time_plan(n, batch, direction, variant, x, y, reps=10, **opts):
    with bf.Plan(n, batch, direction, variant, **opts) as p:
        info = p.info()
        for _ in range(3):
            p.exec(x, y)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            p.exec(x, y)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps, info


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min", type=int, default=8)
    ap.add_argument("--max", type=int, default=22)
    ap.add_argument("--gib", type=float, default=2.0)
    ap.add_argument("--variants", default="1,2,3")
    ap.add_argument("--dirs", default="-1")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    rows = []
    for k in range(a.min, a.max + 1):
        n = 1 << k
        batch = max(1, int(a.gib * 2 ** 30) // (8 * n))
        x = torch.empty((batch, n), dtype=torch.complex64, device="cuda")
        sg.fill_random(x, 1)
        y = torch.empty_like(x)
        for v in [int(t) for t in a.variants.split(",")]:
            cs = [0]
            if v == 2 and k == 16:
                cs = [8, 16]
            for c in cs:
                for d in [int(t) for t in a.dirs.split(",")]:
                    try:
                        ms, info = time_plan(n, batch, d, v, x, y, cluster_size=c)
                    except bf.FFTError as e:
                        continue
                    gbs = 16.0 * n * batch / (ms * 1e-3) / 1e9
                    row = dict(n=n, log2n=k, batch=batch, dir=d, variant=info["variant_name"],
                               cluster=info["cluster"], ms=ms, alg_GBps=gbs, frac=gbs / peak,
                               records_per_s=batch / (ms * 1e-3))
                    rows.append(row)
                    print(f"N=2^{k:<2} {info['variant_name']:>8} C={info['cluster']:<2} dir={d:+d} "
                          f"batch={batch:<8} {ms:8.3f} ms  {gbs:7.1f} GB/s  {gbs / peak:6.1%}  resident={info['resident']}", flush=True)
        del x, y
        torch.cuda.empty_cache()
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
