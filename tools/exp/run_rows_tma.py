# k_rows_tma experiment (tools/exp/exp_rows_tma.cu): 4 GiB of records, rel_l2 vs torch.fft fp64
import ctypes, os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "exp", os.environ.get("EXP_LIB", "librtma.so")))
vp, i32 = ctypes.c_void_p, ctypes.c_int
lib.exp_run.argtypes = [i32, vp, vp, ctypes.c_longlong, i32, ctypes.POINTER(i32)]
lib.exp_run.restype = ctypes.c_float
lib.exp_name.restype = ctypes.c_char_p
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
cfgs = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else range(lib.exp_ncfg())
for i in cfgs:
    n = lib.exp_L(i); b = (4 << 30) // (8 * n)
    x = torch.randn((b, n), dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
    chk = [0, 1, b // 2, b - 1]
    ref = torch.fft.fft(x[chk].to(torch.complex128))
    occ = i32()
    ms = lib.exp_run(i, x.data_ptr(), y.data_ptr(), b, 10, ctypes.byref(occ))
    torch.cuda.synchronize()
    err = float(((y[chk].to(torch.complex128) - ref).abs().pow(2).sum(1).sqrt() / ref.abs().pow(2).sum(1).sqrt()).max())
    gbs = 16.0 * n * b / (ms * 1e-3) / 1e9 if ms > 0 else 0
    print(f"{lib.exp_name(i).decode():26s} occ={occ.value} b={b}: {ms:.3f} ms {gbs:.0f} GB/s ({gbs/peak:.1%}) rel_l2={err:.2e}", flush=True)
    del x, y
