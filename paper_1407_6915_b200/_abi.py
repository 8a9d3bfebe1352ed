"""ctypes binding of include/blockfft.h — argument marshalling only.

Every step of the transform runs in libblockfft.so (CUDA kernels for sm_100a);
this module never computes anything itself and has no CPU fallback: if the
library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libblockfft.so")
STRESS_LIB_PATH = os.path.join(_PKG, "libblockfft_stress.so")

FFT_FORWARD = -1
FFT_INVERSE = +1
FFT_IDENTITY = 0

FFT_OK, FFT_E_SIZE, FFT_E_BATCH, FFT_E_DIR, FFT_E_ARG, FFT_E_DEVICE, FFT_E_CUDA, \
    FFT_E_NOMEM, FFT_E_IO, FFT_E_EMPTY = range(10)
STATUS_NAMES = ["FFT_OK", "FFT_E_SIZE", "FFT_E_BATCH", "FFT_E_DIR", "FFT_E_ARG", "FFT_E_DEVICE",
                "FFT_E_CUDA", "FFT_E_NOMEM", "FFT_E_IO", "FFT_E_EMPTY"]

VARIANT_AUTO, VARIANT_SINGLE, VARIANT_CLUSTER, VARIANT_FOURSTEP, VARIANT_IDENTITY, VARIANT_PIPE = range(6)
VARIANT_NAMES = {0: "auto", 1: "single", 2: "cluster", 3: "fourstep", 4: "identity", 5: "pipe"}

# Every symbol include/blockfft.h declares (checked by tests/test_abi.py).
EXPORTED = ["fft_plan_create", "fft_plan_create_ex", "fft_plan_create_opts", "fft_plan_create_real",
            "fft_plan_create_stft", "fft_exec", "fft_exec_range",
            "fft_plan_destroy", "fft_plan_get_info", "fft_file_records", "fft_partition",
            "fft_file", "fft_file_ex", "fft_file_range", "fft_exec_host", "fft_stream_host",
            "fft_dplan_create", "fft_dplan_exec", "fft_dplan_geometry", "fft_dplan_destroy",
            "fft_numa_node", "fft_host_alloc", "fft_host_free", "fft_link_probe", "fft_stream_release", "fft_last_error", "fft_last_status", "fft_version"]


class PlanInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("batch", ctypes.c_int64), ("dir", ctypes.c_int),
                ("variant", ctypes.c_int), ("kernels_per_exec", ctypes.c_int),
                ("device", ctypes.c_int), ("n1", ctypes.c_int64), ("n2", ctypes.c_int64),
                ("cluster", ctypes.c_int), ("scratch_bytes", ctypes.c_int64),
                ("table_bytes", ctypes.c_int64), ("resident", ctypes.c_int),
                ("exclusive", ctypes.c_int), ("ring_records", ctypes.c_int), ("ring_lag", ctypes.c_int),
                ("real", ctypes.c_int), ("hop", ctypes.c_int64)]


class PlanOpts(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int), ("impl", ctypes.c_int), ("config", ctypes.c_int),
                ("cluster_size", ctypes.c_int), ("ring_records", ctypes.c_int), ("ring_lag", ctypes.c_int)]


class StreamOpts(ctypes.Structure):
    _fields_ = [("chunk_bytes", ctypes.c_int64), ("depth", ctypes.c_int),
                ("variant", ctypes.c_int), ("io_threads", ctypes.c_int),
                ("direct_io", ctypes.c_int), ("numa", ctypes.c_int),
                ("tap_records", ctypes.POINTER(ctypes.c_int64)), ("tap_count", ctypes.c_int64),
                ("tap_out", ctypes.c_void_p), ("timeline", ctypes.POINTER(ctypes.c_double)),
                ("timeline_chunks", ctypes.c_int64), ("real", ctypes.c_int),
                ("hop", ctypes.c_int64), ("window", ctypes.POINTER(ctypes.c_float)),
                ("window_len", ctypes.c_int64)]


TIMELINE_FIELDS = 8
TIMELINE_NAMES = ["read_start", "read_end", "h2d_start", "h2d_end", "fft_end", "d2h_end",
                  "write_start", "write_end"]


class StreamStats(ctypes.Structure):
    _fields_ = [("records", ctypes.c_int64), ("chunks", ctypes.c_int64),
                ("bytes_in", ctypes.c_int64), ("bytes_out", ctypes.c_int64),
                ("wall_s", ctypes.c_double), ("read_s", ctypes.c_double),
                ("h2d_s", ctypes.c_double), ("fft_s", ctypes.c_double),
                ("d2h_s", ctypes.c_double), ("write_s", ctypes.c_double),
                ("ngpu", ctypes.c_int), ("numa_node", ctypes.c_int), ("direct_io", ctypes.c_int),
                ("taps", ctypes.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load a build of the library (default: the product libblockfft.so; tests
    also load the stress build libblockfft_stress.so side by side)."""
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    sig = {
        "fft_plan_create": (vp, [i64, i64, i32]),
        "fft_plan_create_ex": (vp, [i64, i64, i32, i32]),
        "fft_plan_create_opts": (vp, [i64, i64, i32, ctypes.POINTER(PlanOpts)]),
        "fft_plan_create_real": (vp, [i64, i64, i32]),
        "fft_plan_create_stft": (vp, [i64, i64, i64, i32, ctypes.POINTER(ctypes.c_float)]),
        "fft_exec": (i32, [vp, vp, vp, vp]),
        "fft_exec_range": (i32, [vp, vp, vp, i64, vp]),
        "fft_plan_destroy": (None, [vp]),
        "fft_plan_get_info": (i32, [vp, ctypes.POINTER(PlanInfo)]),
        "fft_file_records": (i64, [i64, i64]),
        "fft_partition": (i32, [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "fft_file": (i32, [ctypes.c_char_p, ctypes.c_char_p, i64, i32]),
        "fft_file_ex": (i32, [ctypes.c_char_p, ctypes.c_char_p, i64, i32, i32,
                              ctypes.POINTER(StreamOpts), ctypes.POINTER(StreamStats)]),
        "fft_exec_host": (i32, [i64, i64, i32, vp, vp, i32, ctypes.POINTER(StreamOpts),
                                ctypes.POINTER(StreamStats)]),
        "fft_stream_host": (i32, [i64, i64, i32, vp, i64, vp, i64, i32, ctypes.POINTER(StreamOpts),
                                  ctypes.POINTER(StreamStats)]),
        "fft_file_range": (i32, [ctypes.c_char_p, ctypes.c_char_p, i64, i32, i64, i64, i32,
                                 ctypes.POINTER(StreamOpts), ctypes.POINTER(StreamStats)]),
        "fft_numa_node": (i32, [i32]),
        "fft_dplan_create": (vp, [i64, i32, ctypes.POINTER(i32), i32]),
        "fft_dplan_exec": (i32, [vp, ctypes.POINTER(vp), ctypes.POINTER(vp)]),
        "fft_dplan_geometry": (i32, [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i32)]),
        "fft_dplan_destroy": (None, [vp]),
        "fft_host_alloc": (vp, [i64, i32]),
        "fft_host_free": (None, [vp]),
        "fft_link_probe": (i32, [i32, vp, vp, i64, i32, ctypes.POINTER(ctypes.c_double)]),
        "fft_stream_release": (i32, []),
        "fft_last_error": (ctypes.c_char_p, []),
        "fft_last_status": (i32, []),
        "fft_version": (i32, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = load()
