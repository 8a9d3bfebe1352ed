"""Ring size / lag sweep of the default pipelined plan (experiment tool):
  python tools/exp/sweep_ring.py 16 "0:0,40:20,80:40,..." [gib]   (ring_records:ring_lag, 0 = default)"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import paper_1407_6915_b200 as bf
from synth import gpu as sg
k = int(sys.argv[1]); n = 1 << k
cfgs = [tuple(map(int, c.split(":"))) for c in sys.argv[2].split(",")]
gib = float(sys.argv[3]) if len(sys.argv) > 3 else 4.0
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
b = int(gib * 2 ** 30) // (8 * n)
x = torch.empty((b, n), dtype=torch.complex64, device="cuda"); sg.fill_random(x, 1)
y = torch.empty_like(x)
for S, lag in cfgs:
    with bf.Plan(n, b, -1, bf.VARIANT_PIPE, ring_records=S, ring_lag=lag) as p:
        info = p.info()
        for _ in range(3): p.exec(x, y)
        best = 1e9
        for _ in range(8):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); p.exec(x, y); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
    gbs = 16.0 * n * b / (best * 1e-3) / 1e9
    print(f"N=2^{k} S={info['ring_records']} LAG={info['ring_lag']} {best:7.3f} ms {gbs:7.1f} GB/s {gbs/peak:6.1%}", flush=True)
