"""NEXT-4 timing: one record of n complex64 points over G GPUs (fft_dplan_exec,
the distributed four-step with peer-store transposes), G = 1, 2, 4.  Reports
the wall time of the synchronous call (best of --reps after a warm-up), the
record's points/s, the algorithmic HBM bytes (16 n per pass over HBM... the
record is read and written once: 16 n) over the time, and the NVLink bytes the
three all-to-alls move (3 x 8n (G-1)/G) per GPU per direction over the time.

  python tools/dplan_bench.py [--log2n 30] [--gpus 1,2,4] [--json OUT]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402
from synth import gpu as sg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=30)
    ap.add_argument("--gpus", default="1,2,4")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    n = 1 << a.log2n
    rows = []
    for g in [int(x) for x in a.gpus.split(",")]:
        if g > torch.cuda.device_count():
            rows.append({"gpus": g, "skipped": "not enough GPUs"})
            continue
        per = n // g
        slabs = []
        for i in range(g):
            t = torch.empty(per, dtype=torch.complex64, device=f"cuda:{i}")
            sg.fill_random(t, 7, first_sample=i * per)
            slabs.append(t)
        outs = [torch.empty_like(s) for s in slabs]
        try:
            with bf.DistPlan(n, g) as p:
                p.exec(slabs, outs)
                best = 1e9
                for _ in range(a.reps):
                    t0 = time.perf_counter()
                    p.exec(slabs, outs)
                    best = min(best, time.perf_counter() - t0)
                n1, n2 = p.geometry()
        except bf.FFTError as e:
            rows.append({"gpus": g, "error": str(e)})
            continue
        nv = 3 * 8 * per * (g - 1) / g
        row = {"gpus": g, "n": n, "n1": n1, "n2": n2, "seconds": best, "points_per_s": n / best,
               "alg_GBps_total": 16.0 * n / best / 1e9,
               "nvlink_bytes_per_gpu_each_way": nv, "nvlink_GBps_per_gpu_each_way": nv / best / 1e9}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del slabs, outs
        for i in range(g):
            with torch.cuda.device(i):
                torch.cuda.empty_cache()
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
