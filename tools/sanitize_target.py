"""Small workload for compute-sanitizer: every variant on a few records."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1407_6915_b200 as bf
from synth import gpu as sg
cases = [(1, 1024, 7), (1, 4096, 3), (3, 4096, 3), (2, 1 << 14, 5), (2, 1 << 16, 3), (5, 1 << 14, 9),
         (5, 1 << 16, 5), (5, 1 << 18, 2), (3, 1 << 18, 2)]
for v, n, b in cases:
    for d in (-1, 1):
        x = torch.empty((b, n), dtype=torch.complex64, device="cuda")
        sg.fill_random(x, 3)
        y = torch.empty_like(x)
        with bf.Plan(n, b, d, v) as p:
            p.exec(x, y)
        torch.cuda.synchronize()
        print("ok", v, n, b, d, flush=True)
