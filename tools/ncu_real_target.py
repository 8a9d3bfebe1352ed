"""ncu target: one fused R2C and one fused C2R exec of real records of --n points
(4 GiB of float32 records), for `ncu --set full -k regex:k_rows -c 2`."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
a = ap.parse_args()
floats = (4 << 30) // 4
b = floats // a.n
x = (torch.rand(floats, device="cuda") * 2 - 1).view(b, a.n)
y = torch.empty((b, a.n // 2), dtype=torch.complex64, device="cuda")
with bf.RealPlan(a.n, b, bf.FFT_FORWARD) as p:
    p.exec(x, y)
with bf.RealPlan(a.n, b, bf.FFT_INVERSE) as p:
    p.exec(y, x)
torch.cuda.synchronize()
print("ok")
