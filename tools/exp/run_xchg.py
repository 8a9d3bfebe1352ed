import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
lib = ctypes.CDLL(os.path.join(ROOT, "tools", "exp", "libxchg.so"))
lib.exp_xchg.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.c_int]
lib.exp_xchg.restype = ctypes.c_float
sink = torch.zeros(16, dtype=torch.complex64, device="cuda")
names = ["C=8 NT=256 P=32", "C=16 NT=128 P=32", "C=16 NT=256 P=16", "C=4 NT=256 P=16", "C=8 NT=512 P=16"]
slices = [8192, 4096, 4096, 4096, 8192]
iters = 2000
for vec, vn, reps in ((3, "bulk s2s", 1), (3, "bulk s2s x4", 4), (1, "st.async v2 x4", 4)):
  for i, nm in enumerate(names):
    if vec == 2 and i in (2, 3, 4):
        continue
    ncl = ctypes.c_int()
    ms = lib.exp_xchg(i, vec, iters, sink.data_ptr(), ctypes.byref(ncl), reps)
    nm2 = vn + " " + nm
    us = ms * 1e3 / iters
    # bytes exchanged per iteration across the GPU
    tot = ncl.value * (8 if 'C=8' in nm else 16 if 'C=16' in nm else 4) * slices[i] * 8 * reps
    print(f"{nm2}: clusters={ncl.value} {us:.2f} us/iter  {tot / (us * 1e-6) / 1e12:.2f} TB/s DSMEM (all CTAs)")
