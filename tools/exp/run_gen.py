# k_pipe2 factorisation experiment (tools/exp/exp_gen.cu): N = N1 x N2 at 2^15..2^18; correctness vs torch.fft (context)
import ctypes, os, sys, math, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "exp", os.environ.get("EXP_LIB", "libgen.so")))
vp, i32 = ctypes.c_void_p, ctypes.c_int
lib.exp_run.argtypes = [i32, vp, vp, vp, vp, ctypes.c_longlong, i32, vp, vp, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
lib.exp_run.restype = ctypes.c_float
lib.exp_name.restype = ctypes.c_char_p
assert lib.exp_upload_tw() == 0
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
def tw(m, M):
    m = torch.remainder(torch.as_tensor(m, dtype=torch.float64), M)
    return torch.polar(torch.ones_like(m), -2 * math.pi * m / M).to(torch.complex64).contiguous().cuda()
ar = lambda k: torch.arange(k, dtype=torch.float64)
cfgs = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else range(lib.exp_ncfg())
for i in cfgs:
    n1, n2, pp = lib.exp_n1(i), lib.exp_n2(i), lib.exp_pp(i)
    n = n1 * n2
    b = (4 << 30) // (8 * n)
    x = torch.randn((b, n), dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
    ref = torch.fft.fft(x[:4].to(torch.complex128))
    ta1, tb2 = n1 // pp, n2 // pp
    twm = lib.exp_twm(i)
    lbv = 0
    if twm == 2:     # TW_SPLIT
        wa = tw(ar(ta1).view(-1, 1) * ar(n2).view(1, -1), n)
        wb = torch.cat([tw(ar(tb2).view(-1, 1) * ar(pp).view(1, -1), n2 * pp).flatten(),
                        tw(ar(pp).view(-1, 1) * ar(pp).view(1, -1), pp * pp).flatten()])
    elif twm == 1:   # TW_TABLE: [k1][n2]
        wa = tw(ar(n1).view(-1, 1) * ar(n2).view(1, -1), n); wb = wa
    else:            # TW_TREE: two-level W_N (hi, lo)
        lbv = (n.bit_length() - 1) // 2
        wa = tw(ar(n >> lbv) * (1 << lbv), n); wb = tw(ar(1 << lbv), n)
    maxS = (96 << 20) // (8 * n)
    ring = torch.empty((maxS, n), dtype=torch.complex64, device="cuda")
    ctr = torch.zeros(2 + 2 * maxS, dtype=torch.int32, device="cuda")
    S, occ = i32(), i32()
    ms = lib.exp_run(i, x.data_ptr(), y.data_ptr(), ring.data_ptr(), ctr.data_ptr(), b, maxS,
                     wa.data_ptr(), wb.data_ptr(), lbv, 5, ctypes.byref(S), ctypes.byref(occ))
    torch.cuda.synchronize()
    err = float(((y[:4].to(torch.complex128) - ref).abs().pow(2).sum(1).sqrt() / ref.abs().pow(2).sum(1).sqrt()).max())
    gbs = 16.0 * n * b / (ms * 1e-3) / 1e9 if ms > 0 else 0
    print(f"{lib.exp_name(i).decode():40s} occ={occ.value} S={S.value}: {ms:.3f} ms {gbs:.0f} GB/s ({gbs/peak:.1%}) err={err:.2e}", flush=True)
    del x, y, ring
