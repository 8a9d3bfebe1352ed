"""Time plans with explicit fft_plan_opts (impl, config) per N (experiment tool).
  python tools/exp/sweep_cfg.py 14-20 "2:0,2:2,3:0" [gib]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import paper_1407_6915_b200 as bf
from synth import gpu as sg
lo, hi = map(int, sys.argv[1].split("-"))
cfgs = [tuple(map(int, c.split(":"))) for c in sys.argv[2].split(",")]
gib = float(sys.argv[3]) if len(sys.argv) > 3 else 2.0
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
elems = int(gib * 2 ** 30) // 8
xb = torch.empty(elems, dtype=torch.complex64, device="cuda"); sg.fill_random(xb, 1)
yb = torch.empty_like(xb)
for k in range(lo, hi + 1):
    n = 1 << k; b = elems // n
    x, y = xb[: b * n].view(b, n), yb[: b * n].view(b, n)
    ref = None
    for impl, cfg in cfgs:
        try:
            p = bf.Plan(n, b, -1, bf.VARIANT_PIPE, impl=impl, config=cfg)
        except bf.FFTError as e:
            print(f"N=2^{k} impl={impl} cfg={cfg}: {e}"); continue
        info = p.info()
        for _ in range(3): p.exec(x, y)
        best = 1e9
        for _ in range(8):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); p.exec(x, y); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
        same = ""
        if ref is None: ref = y[:4].clone()
        else: same = "bit-identical" if torch.equal(ref, y[:4]) else "differs"
        p.close()
        gbs = 16.0 * n * b / (best * 1e-3) / 1e9
        print(f"N=2^{k:<2} impl={impl} cfg={cfg} resident={info['resident']} S={info['ring_records']} {best:7.3f} ms {gbs:7.1f} GB/s {gbs/peak:6.1%} {same}", flush=True)
