"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
every variant on a few records, and the pipelined four-step kernels with
batches that wrap their L2 ring (slot reuse: the write-after-read waits, the
L2 discard and the rewrite of a slot) — at the default ring size (2^14, 2^22)
and with the ring forced down to LAG + 1 slots (k_pipe, k_pipe2, k_pipe3).

  compute-sanitizer --tool racecheck python tools/sanitize_target.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402
from synth import gpu as sg  # noqa: E402

quick = "--quick" in sys.argv


def ring_slots(n, **o):
    with bf.Plan(n, 1, **o) as p:
        return p.info()["ring_records"]


# (variant, n, batch, plan options)
cases = [(1, 1024, 7, {}), (1, 4096, 3, {}), (1, 8192, 3, {}), (3, 4096, 3, {}), (2, 1 << 14, 5, {}),
         (2, 1 << 16, 3, {}), (5, 1 << 14, 2 * ring_slots(1 << 14) + 3, {}),
         (5, 1 << 16, 13, dict(ring_lag=3, ring_records=4)),
         (5, 1 << 16, 13, dict(impl=1, ring_lag=3, ring_records=4)),
         (5, 1 << 16, 13, dict(impl=3, ring_lag=3, ring_records=4)),
         (5, 1 << 19, 9, dict(ring_lag=2, ring_records=3)),
         (5, 1 << 22, 2 * ring_slots(1 << 22) + 3, {})]
if quick:
    cases = cases[6:8]
for v, n, b, o in cases:
    for d in (-1, 1):
        x = torch.empty((b, n), dtype=torch.complex64, device="cuda")
        sg.fill_random(x, 3)
        y = torch.empty_like(x)
        with bf.Plan(n, b, d, v, **o) as p:
            p.exec(x, y)
        torch.cuda.synchronize()
        print("ok", v, n, b, d, o, flush=True)
        del x, y
