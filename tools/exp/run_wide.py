# k_pipe2 tile-shape experiment at 2^16 (tools/exp/exp_wide.cu); correctness vs torch.fft (context only)
import ctypes, os, sys, math, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "exp", os.environ.get("EXP_LIB", "libwide.so")))
vp, i32 = ctypes.c_void_p, ctypes.c_int
lib.exp_run.argtypes = [i32, vp, vp, vp, vp, ctypes.c_longlong, i32, vp, vp, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
lib.exp_run.restype = ctypes.c_float
lib.exp_name.restype = ctypes.c_char_p
assert lib.exp_upload_tw() == 0
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
n, b = 65536, 8192
x = torch.randn((b, n), dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
ref = torch.fft.fft(x[:8].to(torch.complex128)).to(torch.complex128)
lb = 8
hi = torch.tensor([complex(math.cos(-2*math.pi*(a<<lb)/n), math.sin(-2*math.pi*(a<<lb)/n)) for a in range(n >> lb)], dtype=torch.complex64, device="cuda")
lo = torch.tensor([complex(math.cos(-2*math.pi*k/n), math.sin(-2*math.pi*k/n)) for k in range(1 << lb)], dtype=torch.complex64, device="cuda")
def tw(m, M):
    m = torch.remainder(torch.as_tensor(m, dtype=torch.float64), M)
    return torch.polar(torch.ones_like(m), -2 * math.pi * m / M).to(torch.complex64).contiguous().cuda()
ar = lambda k: torch.arange(k, dtype=torch.float64)
full = tw(ar(256).view(256, 1) * ar(256).view(1, 256), n)           # TW_TABLE [k1][n2]
one = torch.ones(1, dtype=torch.complex64, device="cuda")
def split_tables(pp):                                                # TW_SPLIT
    ta1 = tb2 = 256 // pp
    wa = tw(ar(ta1).view(-1, 1) * ar(256).view(1, -1), n)
    wb0 = tw(ar(tb2).view(-1, 1) * ar(pp).view(1, -1), 256 * pp)
    t = tw(ar(pp).view(-1, 1) * ar(pp).view(1, -1), pp * pp)
    return wa, torch.cat([wb0.flatten(), t.flatten()])
maxS = (96 << 20) // (8 * n)
ring = torch.empty((maxS, n), dtype=torch.complex64, device="cuda")
ctr = torch.zeros(2 + 2 * maxS, dtype=torch.int32, device="cuda")
cfgs = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else range(lib.exp_ncfg())
for i in cfgs:
    twm, pp = lib.exp_twm(i), lib.exp_pp(i)
    if twm == 1:
        a_, b_, lbv = full, one, 0
    elif twm == 2:
        a_, b_ = split_tables(pp); lbv = 0
    else:
        a_, b_, lbv = hi, lo, lb
    S, occ = i32(), i32()
    y.zero_()
    ms = lib.exp_run(i, x.data_ptr(), y.data_ptr(), ring.data_ptr(), ctr.data_ptr(), b, maxS,
                     a_.data_ptr(), b_.data_ptr(), lbv, 5, ctypes.byref(S), ctypes.byref(occ))
    err = float(((y[:8].to(torch.complex128) - ref).abs().pow(2).sum(1).sqrt() / ref.abs().pow(2).sum(1).sqrt()).max())
    last = float(((torch.fft.fft(x[-2:].to(torch.complex128)) - y[-2:].to(torch.complex128)).abs().max()))
    gbs = 16.0 * n * b / (ms * 1e-3) / 1e9 if ms > 0 else 0
    if hasattr(lib, "exp_prof_read"):
        pr = (ctypes.c_ulonglong * 32)(); lib.exp_prof_read(pr)
        na, nb = max(pr[22], 1), max(pr[23], 1)
        print(f"   per task (cycles, all reps): A wait {pr[18]/na:.0f} work {pr[19]/na:.0f} | B wait {pr[20]/nb:.0f} work {pr[21]/nb:.0f}"
              f" | release: wait done {pr[16]/(na+nb):.0f} fence+red {pr[17]/(na+nb):.0f}")
    print(f"{lib.exp_name(i).decode():32s} occ={occ.value} S={S.value}: {ms:.3f} ms {gbs:.0f} GB/s ({gbs/peak:.1%}) err={err:.2e} lastabs={last:.2e}", flush=True)
