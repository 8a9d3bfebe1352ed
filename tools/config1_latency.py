"""Config 1 (BASELINE.json configs[0]): 16 records x
1024-point complex64, forward — the paper's record length on a
small seeded file.  Latency-bound (no roofline claim): reports the fft_exec
device time (CUDA events, median of 50 after warm-up) and the fft_file wall
time (host clock around the C call, median of 20, file in the page cache),
plus the end-to-end fft_exec_host time from pinned host memory.

  python tools/config1_latency.py [--json OUT]
"""
import argparse
import json
import os
import statistics
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    n, r = 1024, 16
    x_h = synth.random_records(synth.DEFAULT_SEED, n, 0, r)
    x = torch.from_numpy(x_h).cuda()
    y = torch.empty_like(x)
    ev = []
    with bf.Plan(n, r) as p:
        info = p.info()
        for _ in range(10):
            p.exec(x, y)
        torch.cuda.synchronize()
        for _ in range(50):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            p.exec(x, y)
            e.record()
            e.synchronize()
            ev.append(s.elapsed_time(e) * 1e3)
    d = tempfile.mkdtemp()
    src, dst = os.path.join(d, "in.c64"), os.path.join(d, "out.c64")
    x_h.astype("<c8").tofile(src)
    walls = []
    for i in range(25):
        t0 = time.perf_counter()
        bf.fft_file(src, dst, n, 1)
        if i >= 5:
            walls.append((time.perf_counter() - t0) * 1e3)
    h = bf.HostBuffer(r, n, 0)
    o = bf.HostBuffer(r, n, 0)
    h.a[:] = x_h
    host = []
    for i in range(25):
        t0 = time.perf_counter()
        bf.exec_host(h.a, n, bf.FFT_FORWARD, 0, out=o.a)
        if i >= 5:
            host.append((time.perf_counter() - t0) * 1e6)
    assert np.array_equal(o.a, y.cpu().numpy()) and np.array_equal(np.fromfile(dst, "<c8").reshape(r, n), o.a)
    row = {"config": "config1: 16 x 1024-pt complex64 forward, seeded file", "variant": info["variant_name"],
           "fft_exec_us_median": statistics.median(ev), "fft_exec_us_min": min(ev),
           "fft_exec_records_per_s": r / (statistics.median(ev) * 1e-6),
           "fft_file_ms_median": statistics.median(walls), "fft_file_ms_min": min(walls),
           "fft_exec_host_us_median": statistics.median(host),
           "note": "latency case: launch/sync bound, no roofline claim (SURVEY §8(d))"}
    print(json.dumps(row))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(row, f, indent=1)


if __name__ == "__main__":
    main()
