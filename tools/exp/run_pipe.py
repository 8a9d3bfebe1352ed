import ctypes, os, sys, math
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "exp", "libpipe.so"))
vp = ctypes.c_void_p
lib.exp_pipe.argtypes = [vp, vp, vp, vp, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int, vp, vp]
n, b = 65536, 4096
x = torch.randn((b, n), dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
lb = 8
hi = torch.tensor([complex(math.cos(-2*math.pi*(a<<lb)/n), math.sin(-2*math.pi*(a<<lb)/n)) for a in range(n >> lb)], dtype=torch.complex64, device="cuda")
lo = torch.tensor([complex(math.cos(-2*math.pi*k/n), math.sin(-2*math.pi*k/n)) for k in range(1 << lb)], dtype=torch.complex64, device="cuda")
for S, LAG in ((81, 40), (121, 60), (161, 80)):
    ring = torch.empty((S, n), dtype=torch.complex64, device="cuda")
    ctr = torch.zeros(1 + 2 * S, dtype=torch.int32, device="cuda")
    prof = (ctypes.c_ulonglong * 16)(); ms = ctypes.c_float()
    for _ in range(2):
        occ = lib.exp_pipe(x.data_ptr(), y.data_ptr(), ring.data_ptr(), ctr.data_ptr(), b, S, LAG, hi.data_ptr(), lo.data_ptr(), lb, prof, ctypes.byref(ms))
    na, nb = prof[10], prof[11]
    gbs = 16.0 * n * b / (ms.value * 1e-3) / 1e9
    print(f"S={S} LAG={LAG} occ={occ}: {ms.value:.3f} ms {gbs:.0f} GB/s ({gbs/6554.6:.1%}); A tasks {na}, B tasks {nb}")
    print("  A: load+engine %.0f, twiddle %.0f, WAR wait %.0f, store+release %.0f, total %.0f cycles" % tuple(prof[i]/max(na,1) for i in range(5)))
    print("  B: dep wait %.0f, tile load %.0f, engine+store %.0f, total %.0f cycles" % tuple(prof[i]/max(nb,1) for i in range(5, 9)))
