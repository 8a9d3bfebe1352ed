import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "exp", "libdram2.so"))
lib.exp_tile2.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int]
lib.exp_tile2.restype = ctypes.c_float
tot = 1 << 28                       # 2 GiB of complex64 per direction
x = torch.randn(tot, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
for shape, logn in ((0, 16), (1, 20), (2, 22)):
    n = 1 << logn
    b = tot // n
    for mode, name in ((0, "tile rd + tile wr"), (1, "tile rd + flat wr"), (2, "flat rd + tile wr")):
        for w in (4, 8, 16, 32):
            ms = lib.exp_tile2(shape, mode, w, x.data_ptr(), y.data_ptr(), b, 10)
            gbs = 16.0 * n * b / (ms * 1e-3) / 1e9
            print(f"N=2^{logn} {name}: width {w*8:4d} B  {ms:.3f} ms {gbs:7.1f} GB/s {gbs/6554.6:6.1%}", flush=True)
