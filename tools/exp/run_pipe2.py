import ctypes, os, sys, math
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "exp", "libpipe2.so"))
vp = ctypes.c_void_p
lib.exp_pipe2.argtypes = [vp, vp, vp, vp, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int, vp, vp]
n, b = 65536, 4096
x = torch.randn((b, n), dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
lb = 8
hi = torch.tensor([complex(math.cos(-2*math.pi*(a<<lb)/n), math.sin(-2*math.pi*(a<<lb)/n)) for a in range(n >> lb)], dtype=torch.complex64, device="cuda")
lo = torch.tensor([complex(math.cos(-2*math.pi*k/n), math.sin(-2*math.pi*k/n)) for k in range(1 << lb)], dtype=torch.complex64, device="cuda")
for S, LAG in ((140, 60), (121, 60), (124, 55)):
    ring = torch.empty((S, n), dtype=torch.complex64, device="cuda")
    ctr = torch.zeros(1 + 2 * S, dtype=torch.int32, device="cuda")
    prof = (ctypes.c_ulonglong * 32)(); ms = ctypes.c_float()
    occ = lib.exp_pipe2(x.data_ptr(), y.data_ptr(), ring.data_ptr(), ctr.data_ptr(), b, S, LAG, hi.data_ptr(), lo.data_ptr(), lb, prof, ctypes.byref(ms))
    gbs = 16.0 * n * b / (ms.value * 1e-3) / 1e9
    ntask = prof[15]; na, nb = prof[22], prof[23]
    print(f"S={S} LAG={LAG} occ={occ}: {ms.value:.3f} ms {gbs:.0f} GB/s ({gbs/6554.6:.1%}); tasks {ntask} (A {na}, B {nb})")
    print("  producer per task: wait empty %.0f, wait deps %.0f, issue %.0f cycles" % (prof[12]/ntask, prof[13]/ntask, prof[14]/ntask))
    print("  release per task: wait done %.0f, fence+red %.0f" % (prof[16]/ntask, prof[17]/ntask))
    print("  compute A: wait full %.0f, work %.0f | B: wait full %.0f, work %.0f" % (prof[18]/max(na,1), prof[19]/max(na,1), prof[20]/max(nb,1), prof[21]/max(nb,1)))
