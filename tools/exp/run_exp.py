import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
so = os.path.join(ROOT, "tools", "exp", "libexp.so")
import torch
from synth import gpu as sg
lib = ctypes.CDLL(so)
lib.exp_run.argtypes = [ctypes.c_int]*3 + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
n, b = 65536, 4096
x = torch.empty((b, n), dtype=torch.complex64, device="cuda"); sg.fill_random(x, 1)
y = torch.empty_like(x)
peak = 6554.6
for c, mb in ((8, 2), (16, 4), (16, 3)):
    for mode in (0, 1, 2, 3):
        ms = ctypes.c_float()
        ncl = lib.exp_run(c, mb, mode, x.data_ptr(), y.data_ptr(), b, 10, ctypes.byref(ms))
        gbs = 16.0 * n * b / (ms.value * 1e-3) / 1e9
        print(f"C={c:<2} minb={mb} mode={mode} ncl={ncl:<3} {ms.value:.3f} ms {gbs:7.1f} GB/s {gbs/peak:6.1%}", flush=True)
# cuFFT context
for k in (12, 14, 16, 18, 20):
    nn = 1 << k; bb = (1 << 28) // nn
    xx = x.view(-1)[: nn * bb].view(bb, nn)
    torch.fft.fft(xx); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): torch.fft.fft(xx)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    gbs = 16.0 * nn * bb / (ms * 1e-3) / 1e9
    print(f"cuFFT (torch.fft, context only) N=2^{k} batch={bb}: {ms:.3f} ms {gbs:7.1f} GB/s {gbs/peak:6.1%}")
