import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "exp", "libdram.so"))
lib.exp_tile.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int]
lib.exp_tile.restype = ctypes.c_float
n, b = 65536, 4096
x = torch.randn((b, n), dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
for w in (0, 16, 32, 64, 128, 256):
    ms = lib.exp_tile(w, x.data_ptr(), y.data_ptr(), b, 10)
    gbs = 16.0 * n * b / (ms * 1e-3) / 1e9
    print(f"tile width {w*8 if w else 'flat copy'} B: {ms:.3f} ms {gbs:7.1f} GB/s {gbs/6554.6:6.1%}")
