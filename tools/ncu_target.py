"""Minimal launch target for ncu: one plan, `reps` execs on seeded data.

  python tools/ncu_target.py --n 65536 --batch 1024 --variant 2 --reps 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402
from synth import gpu as sg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--dir", type=int, default=-1)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
x = torch.empty((a.batch, a.n), dtype=torch.complex64, device="cuda")
sg.fill_random(x, 1)
y = torch.empty_like(x)
with bf.Plan(a.n, a.batch, a.dir, a.variant) as p:
    print(p.info())
    for _ in range(a.reps):
        p.exec(x, y)
    torch.cuda.synchronize()
print("ok")
