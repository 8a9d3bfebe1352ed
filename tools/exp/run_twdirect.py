# k_pipe2 at 2^16 with the FFT engine compiled out (data movement + sync only) and with deps also removed
import ctypes, os, sys, math
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
vp = ctypes.c_void_p
n, b = 65536, 8192
x = torch.randn((b, n), dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
lb = 8
hi = torch.tensor([complex(math.cos(-2*math.pi*(a<<lb)/n), math.sin(-2*math.pi*(a<<lb)/n)) for a in range(n >> lb)], dtype=torch.complex64, device="cuda")
lo = torch.tensor([complex(math.cos(-2*math.pi*k/n), math.sin(-2*math.pi*k/n)) for k in range(1 << lb)], dtype=torch.complex64, device="cuda")
for name in ("libnc_base.so", "libnc_twdirect.so", "libnc_base.so", "libnc_twdirect.so"):
    lib = ctypes.CDLL(os.path.join(ROOT, "tools", "exp", name))
    lib.exp_run.argtypes = [vp, vp, vp, vp, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int]
    lib.exp_run.restype = ctypes.c_float
    for S, LAG in ((131, 56),):
        ring = torch.empty((S, n), dtype=torch.complex64, device="cuda")
        ctr = torch.zeros(1 + 2 * S, dtype=torch.int32, device="cuda")
        ms = lib.exp_run(x.data_ptr(), y.data_ptr(), ring.data_ptr(), ctr.data_ptr(), b, S, LAG, hi.data_ptr(), lo.data_ptr(), lb)
        gbs = 16.0 * n * b / (ms * 1e-3) / 1e9
        print(f"{name} S={S} LAG={LAG}: {ms:.3f} ms {gbs:.0f} GB/s ({gbs/6554.6:.1%})", flush=True)
