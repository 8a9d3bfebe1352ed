"""Real-record (R2C / C2R) throughput in HBM: RealPlan over --gib GiB of float32
records per N, forward and inverse; algorithmic bytes 8N per real record (4N
in, 4N out); CUDA events, best of 10 after warm-up.
  python tools/real_bench.py [--gib 4] [--json OUT]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gib", type=float, default=4.0)
ap.add_argument("--json", default=None)
a = ap.parse_args()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
rows = []
floats = int(a.gib * 2 ** 30) // 4
buf = torch.rand(floats, device="cuda") * 2 - 1
out = torch.empty(floats // 2, dtype=torch.complex64, device="cuda")
import os
KS = [int(v) for v in os.environ.get("REAL_BENCH_K", "10,12,13,14,15,16,18,20").split(",")]
for k in KS:
    n = 1 << k
    b = floats // n
    x, y = buf[: b * n].view(b, n), out[: b * n // 2].view(b, n // 2)
    for d in (bf.FFT_FORWARD, bf.FFT_INVERSE):
        with bf.RealPlan(n, b, d) as p:
            src, dst = (x, y) if d == bf.FFT_FORWARD else (y, x.clone() if False else x)
            for _ in range(3):
                p.exec(src, dst)
            best = 1e9
            for _ in range(10):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(); p.exec(src, dst); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
            kpe = p.info()["kernels_per_exec"]
        gbs = 8.0 * n * b / (best * 1e-3) / 1e9
        row = {"n": n, "dir": d, "batch": b, "ms": best, "alg_GBps": gbs, "frac": gbs / peak, "kernels": kpe,
               "records_per_s": b / (best * 1e-3)}
        rows.append(row)
        print(f"real N=2^{k:<2} dir={d:+d} batch={b:<8} {best:7.3f} ms {gbs:7.1f} GB/s {gbs/peak:6.1%} kernels={kpe}",
              flush=True)
if a.json:
    json.dump(rows, open(a.json, "w"), indent=1)
