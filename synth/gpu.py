"""CUDA fill of the seeded generator (synth/csrc/synth_fill.cu via ctypes).

Bit-identical to ``synth.random_samples``; used to create multi-GiB benchmark
inputs directly in HBM.  Holds none of the method's arithmetic."""
from __future__ import annotations

import ctypes
import os

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing; run __graft_entry__.build()")
        lib = ctypes.CDLL(_LIB)
        lib.synth_fill_random.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_uint64, ctypes.c_void_p]
        lib.synth_fill_random.restype = ctypes.c_int
        _lib = lib
    return _lib


def fill_random(t, seed: int, first_sample: int = 0, stream=None):
    """Fill complex64 CUDA tensor ``t`` with global samples
    [first_sample, first_sample + t.numel()) of stream ``seed``."""
    import torch
    assert t.is_cuda and t.dtype == torch.complex64 and t.is_contiguous()
    with torch.cuda.device(t.device):     # launch on the tensor's own GPU
        s = stream if stream is not None else torch.cuda.current_stream(t.device)
        rc = _load().synth_fill_random(ctypes.c_void_p(t.data_ptr()), int(first_sample), t.numel(),
                                       ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"synth_fill_random failed: cudaError {rc}")
    return t
