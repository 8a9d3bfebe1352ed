"""ncu target for the config-5 DRAM sweep: one warm-up and one measured
fft_exec of the default plan per N (forward), 4 GiB of records per N.
Run under `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum`
(tools/sweep.py --ncu-csv parses the result)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402
from synth import gpu as sg  # noqa: E402

lo, hi = int(sys.argv[1]) if len(sys.argv) > 1 else 8, int(sys.argv[2]) if len(sys.argv) > 2 else 22
buf_in = torch.empty(1 << 29, dtype=torch.complex64, device="cuda")   # 4 GiB
buf_out = torch.empty_like(buf_in)
sg.fill_random(buf_in, 1)
for k in range(lo, hi + 1):
    n = 1 << k
    b = (1 << 29) // n
    x, y = buf_in.view(b, n), buf_out.view(b, n)
    with bf.Plan(n, b) as p:
        p.exec(x, y)
        p.exec(x, y)
    torch.cuda.synchronize()
    print(f"N=2^{k} batch={b}", flush=True)
