"""CPU double-precision oracle for the per-record FFT of arXiv 1407.6915.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product path (``paper_1407_6915_b200``) never imports it and
shares no code, header, table or constant with it.

The arithmetic lives in ``oracle.c`` (plain C, fp64, no fast-math):

* ``dft``  – the O(N^2) direct definition, any N >= 1;
* ``fft``  – the textbook recursive radix-2 Cooley–Tukey FFT
  (§I; north_star), N a power of two.

Both follow the conventions of DESIGN.md readings c2/c3: forward
``X[k] = sum_j x[j] e^{-2 pi i jk/N}`` unnormalised, inverse scaled by 1/N
(SPEC.md:36, :75, :90).

File-level semantics (``file_transform``): the input is split into records of
N complex64 samples in file order, the final record zero-padded (reading c6,
SPEC.md:124, :188), every record transformed independently (PAPER.md:49-53
§III) and the outputs concatenated in file order (§III, "named by
their position in the original file"; reading c5).

Parity: pinned by closed forms, brute force, Parseval / linearity /
round-trip / shift / Hermitian invariants and a numpy.fft cross-check in
``tests/test_oracle.py`` — no function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

FORWARD = -1
INVERSE = +1


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc -O2 -fopenmp, no fast-math)."""
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)):
        return _LIB_PATH
    cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
           "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", _LIB_PATH + ".tmp", "-lm"]
    subprocess.check_call(cmd)
    os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        lib.oracle_dft.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int]
        lib.oracle_dft.restype = ctypes.c_int
        lib.oracle_fft.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int]
        lib.oracle_fft.restype = ctypes.c_int
        lib.oracle_batch_c64.argtypes = [fp, dp, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.oracle_batch_c64.restype = ctypes.c_int
        lib.oracle_max_threads.argtypes = []
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _one(fn, x, direction):
    lib = _load()
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    if x.ndim != 1:
        raise ValueError("expected a 1-D record")
    out = np.empty_like(x)
    rc = getattr(lib, fn)(_dptr(x.view(np.float64)), _dptr(out.view(np.float64)),
                          x.shape[0], int(direction))
    if rc != 0:
        raise ValueError(f"{fn}: invalid arguments (n={x.shape[0]}, dir={direction})")
    return out


def dft(x, direction: int = FORWARD) -> np.ndarray:
    """Direct O(N^2) DFT of one record (complex128 in, complex128 out)."""
    return _one("oracle_dft", x, direction)


def fft(x, direction: int = FORWARD) -> np.ndarray:
    """Recursive radix-2 FFT of one record, N a power of two."""
    return _one("oracle_fft", x, direction)


def records_c64(x, direction: int = FORWARD, algo: str = "fft",
                threads: int = 0) -> np.ndarray:
    """Transform each row of a [B, N] complex64 array independently.

    The complex64 values are promoted exactly to double; the result is
    complex128 [B, N].  ``algo`` is ``"fft"`` (recursive radix-2) or ``"dft"``.
    """
    lib = _load()
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex64))
    if x.ndim != 2:
        raise ValueError("expected (B, N) complex64")
    b, n = x.shape
    out = np.empty((b, n), dtype=np.complex128)
    rc = lib.oracle_batch_c64(
        x.view(np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
        _dptr(out.view(np.float64)), n, b, int(direction),
        0 if algo == "fft" else 1, int(threads))
    if rc != 0:
        raise ValueError(f"oracle batch failed (n={n}, algo={algo}, dir={direction})")
    return out


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def pad_records(samples, n: int) -> np.ndarray:
    """Split a flat complex64 sample stream into [R, n] records, R = ceil(len/n),
    zero-padding the final record (reading c6)."""
    s = np.asarray(samples, dtype=np.complex64).reshape(-1)
    if s.size == 0:
        raise ValueError("empty input")
    r = -(-s.size // n)
    out = np.zeros(r * n, dtype=np.complex64)
    out[: s.size] = s
    return out.reshape(r, n)


def file_transform(raw: bytes, n: int, direction: int = FORWARD,
                   threads: int = 0) -> np.ndarray:
    """File-level oracle: headerless little-endian complex64 bytes → [R, n]
    complex128 transforms in file order (§III)."""
    if len(raw) % 8:
        raise ValueError(f"file size {len(raw)} is not a multiple of 8 bytes")
    samples = np.frombuffer(raw, dtype="<c8")
    return records_c64(pad_records(samples, n), direction, "fft", threads)


def rel_l2(y, ref) -> np.ndarray:
    """Per-record relative L2 error ||y - ref|| / ||ref|| in double (§8(c) 5).
    A record whose reference is exactly zero gets error 0 iff y is exactly
    zero, else +inf."""
    y = np.asarray(y, dtype=np.complex128)
    ref = np.asarray(ref, dtype=np.complex128)
    if y.ndim == 1:
        y, ref = y[None], ref[None]
    num = np.sqrt(np.sum(np.abs(y - ref) ** 2, axis=1))
    den = np.sqrt(np.sum(np.abs(ref) ** 2, axis=1))
    out = np.empty(num.shape)
    zero = den == 0
    out[~zero] = num[~zero] / den[~zero]
    out[zero] = np.where(num[zero] == 0, 0.0, np.inf)
    return out


def tolerance(n: int) -> float:
    """north_star bar: relative L2 <= 1e-5 * log2(N) per record (reading c10).
    N = 1 is not a supported transform; for completeness its bar is 1e-5."""
    return 1e-5 * max(1.0, float(np.log2(n)))
