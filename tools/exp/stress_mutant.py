"""Sensitivity check of tests/test_gpu_stress.py (mutation experiment): run the
stress comparison against a library built with a protocol wait REMOVED
(-DBFFT_PIPE_NOWAR: no write-after-read wait before an A-task rewrites a ring
slot; -DBFFT_PIPE_NODEPS: no dependency waits at all) and report how many
records differ from the product build.  A sound check must see differences.
  python tools/exp/stress_mutant.py tools/exp/libmut_nowar.so ..."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402
from paper_1407_6915_b200 import _abi  # noqa: E402
from synth import gpu as sg  # noqa: E402

for path in sys.argv[1:]:
    lib = _abi.load(path)
    for n, b, o in ((1 << 14, None, {}), (1 << 16, 17, dict(ring_lag=3, ring_records=4)),
                    (1 << 16, 301, {}), (1 << 20, 9, dict(ring_lag=2, ring_records=3)), (1 << 22, None, {})):
        if b is None:
            with bf.Plan(n, 1, **o) as p:
                b = 2 * p.info()["ring_records"] + 3
        x = torch.empty((b, n), dtype=torch.complex64, device="cuda")
        sg.fill_random(x, 5 + n)
        ref = torch.empty_like(x)
        with bf.Plan(n, b, -1, bf.VARIANT_PIPE, impl=2, **o) as p:
            p.exec(x, ref)
        torch.cuda.synchronize()
        bad = 0
        for rep in range(3):
            y = torch.full_like(x, float("nan"))
            opts = _abi.PlanOpts(bf.VARIANT_PIPE, 2, 0, 0, o.get("ring_records", 0), o.get("ring_lag", 0))
            h = lib.fft_plan_create_opts(n, b, -1, ctypes.byref(opts))
            lib.fft_exec(ctypes.c_void_p(h), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            torch.cuda.synchronize()
            lib.fft_plan_destroy(ctypes.c_void_p(h))
            bad += int((y.view(torch.float32) != ref.view(torch.float32)).view(b, -1).any(dim=1).sum())
        print(f"{os.path.basename(path)} N=2^{n.bit_length() - 1} batch={b} {o}: {bad} records differ over 3 runs",
              flush=True)
        del x, ref, y
        torch.cuda.empty_cache()
