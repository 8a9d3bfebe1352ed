# k_tri experiment (tools/exp/exp_tri.cu): correctness vs torch.fft (fp64) and timing; args: cfg list, then S,L1,L2 triples
import ctypes, os, sys, math, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "exp", os.environ.get("EXP_LIB", "libtri.so")))
vp, i32 = ctypes.c_void_p, ctypes.c_int
lib.exp_run.argtypes = [i32, vp, vp, vp, vp, ctypes.c_longlong, i32, i32, i32, vp, vp, i32, i32]
lib.exp_run.restype = ctypes.c_float
lib.exp_name.restype = ctypes.c_char_p
assert lib.exp_upload_tw() == 0
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
cfgs = [int(a) for a in sys.argv[1].split(",")]
trip = [tuple(int(v) for v in a.split(",")) for a in sys.argv[2:]] or [(3, 1, 2)]
for i in cfgs:
    lg = lib.exp_logn(i); n = 1 << lg
    b = (4 << 30) // (8 * n)
    x = torch.randn((b, n), dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
    lb = 11
    ar = torch.arange(n >> lb, dtype=torch.float64) * (1 << lb)
    hi = torch.polar(torch.ones_like(ar), -2 * math.pi * ar / n).to(torch.complex64).cuda()
    al = torch.arange(1 << lb, dtype=torch.float64)
    lo = torch.polar(torch.ones_like(al), -2 * math.pi * al / n).to(torch.complex64).cuda()
    chk = [0, 1, b // 2, b - 1]
    ref = torch.fft.fft(x[chk].to(torch.complex128))
    for (S, L1, L2) in trip:
        ring = torch.empty((S, n), dtype=torch.complex64, device="cuda")
        ctr = torch.zeros(lib.exp_nctr(i, S), dtype=torch.int32, device="cuda")
        y.zero_()
        ms = lib.exp_run(i, x.data_ptr(), y.data_ptr(), ring.data_ptr(), ctr.data_ptr(), b, S, L1, L2,
                         hi.data_ptr(), lo.data_ptr(), lb, 5)
        torch.cuda.synchronize()
        err = float(((y[chk].to(torch.complex128) - ref).abs().pow(2).sum(1).sqrt() / ref.abs().pow(2).sum(1).sqrt()).max())
        left = int(ctr.abs().sum())
        gbs = 16.0 * n * b / (ms * 1e-3) / 1e9 if ms > 0 else 0
        print(f"{lib.exp_name(i).decode():24s} b={b} S={S} L1={L1} L2={L2}: {ms:.3f} ms {gbs:.0f} GB/s ({gbs/peak:.1%}) rel_l2={err:.2e} ctr_left={left}", flush=True)
        del ring
