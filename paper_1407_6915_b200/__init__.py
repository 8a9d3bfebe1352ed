"""paper_1407_6915_b200 — B200-native per-record FFT over very large signal files
(arXiv 1407.6915, "Accelerating Fast Fourier Transforms Using Hadoop and CUDA").

Thin Python layer over the C ABI in ``include/blockfft.h`` (``libblockfft.so``):
argument marshalling only; every step of the transform runs in the library's
sm_100a kernels.  PyTorch is used for device memory and streams.

    import paper_1407_6915_b200 as bf
    plan = bf.Plan(n=65536, batch=8192)          # fft_plan_create
    plan.exec(x, y)                              # fft_exec on the current stream
    bf.fft_file("in.c64", "out.c64", 1024, ngpu=2)   # the whole method on a file
"""
from __future__ import annotations

import ctypes
import os

from . import _abi
from ._abi import (FFT_FORWARD, FFT_IDENTITY, FFT_INVERSE, VARIANT_AUTO, VARIANT_CLUSTER,  # noqa: F401
                   VARIANT_FOURSTEP, VARIANT_IDENTITY, VARIANT_NAMES, VARIANT_PIPE, VARIANT_SINGLE)

_lib = _abi.lib


class FFTError(RuntimeError):
    """A libblockfft call failed; ``code`` is the FFT_E_* status."""

    def __init__(self, code: int, msg: str):
        self.code = code
        name = _abi.STATUS_NAMES[code] if 0 <= code < len(_abi.STATUS_NAMES) else str(code)
        super().__init__(f"{name}: {msg}")


def last_error() -> str:
    return (_lib.fft_last_error() or b"").decode()


def _check(rc: int):
    if rc != 0:
        raise FFTError(rc, last_error())


def version() -> int:
    return int(_lib.fft_version())


class Plan:
    """Batched plan: ``batch`` records of ``n`` complex64 points (fft_plan_create).

    Bound to the CUDA device current at construction.  ``exec`` enqueues on the
    current torch stream (or ``stream``) and returns immediately.
    """

    def __init__(self, n: int, batch: int, direction: int = FFT_FORWARD,
                 variant: int = VARIANT_AUTO, device=None, *, impl: int = 0, config: int = 0,
                 cluster_size: int = 0, ring_records: int = 0, ring_lag: int = 0):
        """``impl``, ``config``, ``cluster_size``, ``ring_records``, ``ring_lag``
        are the fft_plan_opts fields (0 = the shipped default for n)."""
        import torch
        self.n, self.batch, self.direction = int(n), int(batch), int(direction)
        if device is not None:
            torch.cuda.set_device(device)
        self.device = torch.cuda.current_device() if torch.cuda.is_available() else None
        opts = _abi.PlanOpts(int(variant), int(impl), int(config), int(cluster_size), int(ring_records),
                             int(ring_lag))
        h = _lib.fft_plan_create_opts(self.n, self.batch, self.direction, ctypes.byref(opts))
        if not h:
            raise FFTError(int(_lib.fft_last_status()), last_error())
        self._h = ctypes.c_void_p(h)

    def info(self) -> dict:
        inf = _abi.PlanInfo()
        _check(_lib.fft_plan_get_info(self._h, ctypes.byref(inf)))
        d = {name: getattr(inf, name) for name, _ in inf._fields_}
        d["variant_name"] = VARIANT_NAMES.get(d["variant"], "?")
        return d

    def _validate(self, t, name, count):
        import torch
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch.Tensor")
        if t.dtype != torch.complex64:
            raise ValueError(f"{name}: expected dtype complex64, got {t.dtype}")
        if not t.is_cuda:
            raise ValueError(f"{name}: expected a CUDA tensor")
        if t.device.index != self.device:
            raise ValueError(f"{name}: expected a tensor on cuda:{self.device} (the plan's device), "
                             f"got {t.device}")
        if not t.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous tensor")
        if t.numel() != count * self.n or (t.dim() == 2 and tuple(t.shape) != (count, self.n)):
            raise ValueError(f"{name}: expected (B,N)=({count},{self.n}) got {tuple(t.shape)}")

    def exec(self, x, out=None, stream=None, count: int | None = None):
        """Transform ``count`` (default: batch) records of x into out (default:
        in place).  Returns out."""
        import torch
        count = self.batch if count is None else int(count)
        if out is None:
            out = x
        self._validate(x, "input", count)
        self._validate(out, "output", count)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = _lib.fft_exec_range(self._h, ctypes.c_void_p(x.data_ptr()),
                                 ctypes.c_void_p(out.data_ptr()), count,
                                 ctypes.c_void_p(s.cuda_stream))
        _check(rc)
        return out

    __call__ = exec

    def close(self):
        if getattr(self, "_h", None):
            _lib.fft_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class RealPlan(Plan):
    """Batched transform of real records (fft_plan_create_real): forward maps
    (B, n) float32 -> (B, n/2) complex64 packed half spectra (out[:, 0] =
    (X[0], X[n/2]), out[:, k] = X[k]); inverse maps them back, scaled by 1/n."""

    def __init__(self, n: int, batch: int, direction: int = FFT_FORWARD, device=None):
        import torch
        self.n, self.batch, self.direction = int(n), int(batch), int(direction)
        if device is not None:
            torch.cuda.set_device(device)
        self.device = torch.cuda.current_device() if torch.cuda.is_available() else None
        h = _lib.fft_plan_create_real(self.n, self.batch, self.direction)
        if not h:
            raise FFTError(int(_lib.fft_last_status()), last_error())
        self._h = ctypes.c_void_p(h)

    def _check_real(self, t, name, count, real):
        import torch
        want = (torch.float32, self.n) if real else (torch.complex64, self.n // 2)
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch.Tensor")
        if t.dtype != want[0]:
            raise ValueError(f"{name}: expected dtype {want[0]}, got {t.dtype}")
        if not t.is_cuda or t.device.index != self.device:
            raise ValueError(f"{name}: expected a tensor on cuda:{self.device}, got {t.device}")
        if not t.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous tensor")
        if t.numel() != count * want[1] or (t.dim() == 2 and tuple(t.shape) != (count, want[1])):
            raise ValueError(f"{name}: expected (B,N)=({count},{want[1]}) got {tuple(t.shape)}")

    def exec(self, x, out=None, stream=None, count: int | None = None):
        import torch
        count = self.batch if count is None else int(count)
        fwd = self.direction == FFT_FORWARD
        if out is None:
            out = torch.empty((count, self.n // 2) if fwd else (count, self.n),
                              dtype=torch.complex64 if fwd else torch.float32, device=x.device)
        self._check_real(x, "input", count, real=fwd)
        self._check_real(out, "output", count, real=not fwd)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(_lib.fft_exec_range(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                   count, ctypes.c_void_p(s.cuda_stream)))
        return out

    __call__ = exec


class StftPlan(Plan):
    """Short-time Fourier transform (fft_plan_create_stft): ``frames`` frames of
    n samples every ``hop`` samples of a complex64 signal, times an optional
    real window; exec(signal, out) with signal of (frames-1)*hop + n samples
    and out (frames, n)."""

    def __init__(self, n: int, hop: int, frames: int, direction: int = FFT_FORWARD, window=None, device=None):
        import numpy as np
        import torch
        self.n, self.batch, self.direction, self.hop = int(n), int(frames), int(direction), int(hop)
        if device is not None:
            torch.cuda.set_device(device)
        self.device = torch.cuda.current_device() if torch.cuda.is_available() else None
        w = None
        if window is not None:
            self._win = np.ascontiguousarray(np.asarray(window, dtype=np.float32))
            if self._win.shape != (self.n,):
                raise ValueError(f"window: expected ({self.n},) got {self._win.shape}")
            w = self._win.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        h = _lib.fft_plan_create_stft(self.n, self.hop, self.batch, self.direction, w)
        if not h:
            raise FFTError(int(_lib.fft_last_status()), last_error())
        self._h = ctypes.c_void_p(h)

    def exec(self, x, out=None, stream=None, count: int | None = None):
        import torch
        count = self.batch if count is None else int(count)
        need = (count - 1) * self.hop + self.n
        if x.dtype != torch.complex64 or not x.is_cuda or not x.is_contiguous() or x.numel() < need:
            raise ValueError(f"input: expected a contiguous complex64 CUDA signal of >= {need} samples")
        if out is None:
            out = torch.empty((count, self.n), dtype=torch.complex64, device=x.device)
        self._validate(out, "output", count)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(_lib.fft_exec_range(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                   count, ctypes.c_void_p(s.cuda_stream)))
        return out

    __call__ = exec


class DistPlan:
    """One record larger than a GPU (fft_dplan_create): n complex64 points as
    ``ngpu`` contiguous slabs, slab g on device ``devices[g]``; exec(slabs_in,
    slabs_out) transforms in natural order (synchronous)."""

    def __init__(self, n: int, ngpu: int, direction: int = FFT_FORWARD, devices=None):
        self.n, self.ngpu, self.direction = int(n), int(ngpu), int(direction)
        self.devices = list(devices) if devices is not None else list(range(self.ngpu))
        arr = (ctypes.c_int * self.ngpu)(*self.devices)
        h = _lib.fft_dplan_create(self.n, self.ngpu, arr, self.direction)
        if not h:
            raise FFTError(int(_lib.fft_last_status()), last_error())
        self._h = ctypes.c_void_p(h)

    def geometry(self) -> tuple[int, int]:
        n1, n2, g = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        _check(_lib.fft_dplan_geometry(self._h, ctypes.byref(n1), ctypes.byref(n2), ctypes.byref(g)))
        return n1.value, n2.value

    def exec(self, slabs_in, slabs_out=None):
        import torch
        slabs_out = slabs_in if slabs_out is None else slabs_out
        per = self.n // self.ngpu
        for g, (a, b) in enumerate(zip(slabs_in, slabs_out)):
            for t in (a, b):
                if t.dtype != torch.complex64 or not t.is_contiguous() or t.numel() != per or \
                        t.device != torch.device("cuda", self.devices[g]):
                    raise ValueError(f"slab {g}: expected {per} contiguous complex64 on cuda:{self.devices[g]}")
        pin = (ctypes.c_void_p * self.ngpu)(*[t.data_ptr() for t in slabs_in])
        pout = (ctypes.c_void_p * self.ngpu)(*[t.data_ptr() for t in slabs_out])
        _check(_lib.fft_dplan_exec(self._h, pin, pout))
        return slabs_out

    def close(self):
        if getattr(self, "_h", None):
            _lib.fft_dplan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def fft(x, direction: int = FFT_FORWARD, variant: int = VARIANT_AUTO, out=None):
    """One-shot batched FFT of a (B, N) complex64 CUDA tensor (plan per call)."""
    b, n = x.shape
    with Plan(n, b, direction, variant) as p:
        if out is None:
            import torch
            out = torch.empty_like(x)
        p.exec(x, out)
        import torch
        torch.cuda.current_stream().synchronize()
    return out


class StreamOptions:
    """fft_stream_opts (include/blockfft.h) with Python-owned tap and timeline
    buffers.  ``taps``: record indices whose outputs are captured (``tap_out``
    after the call, shape (len(taps), n) complex64); ``timeline``: number of
    chunks to record (``timeline_out``, shape (chunks, 8) float64 seconds)."""

    def __init__(self, n=0, chunk_bytes=0, depth=0, variant=VARIANT_AUTO, io_threads=0, direct_io=False,
                 numa=True, taps=None, timeline=0, real=False, hop=0, window=None):
        import numpy as np
        self.c = _abi.StreamOpts()
        self.c.real = int(bool(real))
        self.c.hop = int(hop)
        self.window = None
        if window is not None:
            self.window = np.ascontiguousarray(np.asarray(window, dtype=np.float32))
            self.c.window = self.window.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
            self.c.window_len = self.window.size
        self.c.chunk_bytes, self.c.depth, self.c.variant = int(chunk_bytes), int(depth), int(variant)
        self.c.io_threads, self.c.direct_io, self.c.numa = int(io_threads), int(bool(direct_io)), 0 if numa else -1
        self.tap_records = self.tap_out = self.timeline_out = None
        if taps is not None and len(taps):
            self.tap_records = np.ascontiguousarray(np.asarray(taps, dtype=np.int64))
            self.tap_out = np.zeros((len(self.tap_records), int(n) // 2 if real else int(n)), dtype=np.complex64)
            self.c.tap_records = self.tap_records.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
            self.c.tap_count = len(self.tap_records)
            self.c.tap_out = self.tap_out.ctypes.data
        if timeline:
            self.timeline_out = np.full((int(timeline), _abi.TIMELINE_FIELDS), np.nan)
            self.c.timeline = self.timeline_out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
            self.c.timeline_chunks = int(timeline)


def _opts(chunk_bytes=0, depth=0, variant=VARIANT_AUTO, io_threads=0, options=None):
    if options is not None:
        return options.c
    return StreamOptions(chunk_bytes=chunk_bytes, depth=depth, variant=variant, io_threads=io_threads).c


def fft_file(in_path: str, out_path: str, record_len: int, ngpu: int = 1,
             direction: int = FFT_FORWARD, chunk_bytes: int = 0, depth: int = 0,
             variant: int = VARIANT_AUTO, options: StreamOptions | None = None) -> dict:
    """The whole method on a file (fft_file_ex).  Returns the stream stats."""
    st = _abi.StreamStats()
    o = _opts(chunk_bytes, depth, variant, options=options)
    rc = _lib.fft_file_ex(os.fsencode(in_path), os.fsencode(out_path), int(record_len), int(ngpu),
                          int(direction), ctypes.byref(o), ctypes.byref(st))
    _check(rc)
    return st.as_dict()


def file_range(in_path: str, out_path: str, record_len: int, first: int, count: int, device: int = 0,
               direction: int = FFT_FORWARD, options: StreamOptions | None = None) -> dict:
    """One GPU's share of a file (fft_file_range): records [first, first+count)
    written at their own offsets of out_path (not truncated, not renamed)."""
    st = _abi.StreamStats()
    o = _opts(options=options)
    rc = _lib.fft_file_range(os.fsencode(in_path), os.fsencode(out_path), int(record_len), int(direction),
                             int(first), int(count), int(device), ctypes.byref(o), ctypes.byref(st))
    _check(rc)
    return st.as_dict()


def exec_host(x_host, n: int, direction: int = FFT_FORWARD, device: int = 0, out=None,
              chunk_bytes: int = 0, depth: int = 0, variant: int = VARIANT_AUTO,
              options: StreamOptions | None = None) -> dict:
    """Transform records held in host memory (torch CPU tensor, pinned or not,
    or numpy array) through the streamer (fft_exec_host).  In place unless
    ``out`` is given.  Returns the stream stats."""
    if out is None:
        out = x_host
    ptr_in, nbytes = _host_ptr(x_host)
    ptr_out, nbytes_o = _host_ptr(out)
    rb = (4 if options is not None and options.c.real else 8) * n
    if nbytes != nbytes_o or nbytes % rb:
        raise ValueError(f"expected equal host buffers of a multiple of {rb} bytes, got {nbytes} / {nbytes_o}")
    st = _abi.StreamStats()
    o = _opts(chunk_bytes, depth, variant, options=options)
    rc = _lib.fft_exec_host(int(n), nbytes // rb, int(direction), ctypes.c_void_p(ptr_in),
                            ctypes.c_void_p(ptr_out), int(device), ctypes.byref(o), ctypes.byref(st))
    _check(rc)
    return st.as_dict()


def stream_host(x_ring, out_ring, n: int, total_records: int, direction: int = FFT_FORWARD, device: int = 0,
                options: StreamOptions | None = None) -> dict:
    """fft_stream_host: a logical stream of ``total_records`` records read from
    the host ring ``x_ring`` (record r from ring record r mod len) and written
    to the host ring ``out_ring``.  Returns the stream stats."""
    ptr_in, nb_in = _host_ptr(x_ring)
    ptr_out, nb_out = _host_ptr(out_ring)
    rb = (4 if options is not None and options.c.real else 8) * n
    if nb_in % rb or nb_out % rb:
        raise ValueError(f"ring sizes must be multiples of {rb} bytes, got {nb_in} / {nb_out}")
    st = _abi.StreamStats()
    o = _opts(options=options)
    rc = _lib.fft_stream_host(int(n), int(total_records), int(direction), ctypes.c_void_p(ptr_in),
                              nb_in // rb, ctypes.c_void_p(ptr_out), nb_out // rb, int(device),
                              ctypes.byref(o), ctypes.byref(st))
    _check(rc)
    return st.as_dict()


def numa_node(device: int) -> int:
    return int(_lib.fft_numa_node(int(device)))


class HostBuffer:
    """Pinned host memory on a GPU's NUMA node (fft_host_alloc), exposed as a
    numpy complex64 array ``a`` of shape (records, n)."""

    def __init__(self, records: int, n: int, device: int = 0):
        import numpy as np
        nbytes = int(records) * 8 * int(n)
        p = _lib.fft_host_alloc(nbytes, int(device))
        if not p:
            raise FFTError(int(_lib.fft_last_status()), last_error())
        self._p = p
        self.a = np.ctypeslib.as_array((ctypes.c_char * nbytes).from_address(p)).view(np.complex64).reshape(
            int(records), int(n))

    def close(self):
        if getattr(self, "_p", None):
            self.a = None
            _lib.fft_host_free(ctypes.c_void_p(self._p))
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def link_probe(device: int, src: HostBuffer, dst: HostBuffer, nbytes: int, reps: int = 3) -> dict:
    """fft_link_probe: H2D / D2H GB/s alone and concurrently (pinned buffers)."""
    g = (ctypes.c_double * 5)()
    _check(_lib.fft_link_probe(int(device), ctypes.c_void_p(src._p), ctypes.c_void_p(dst._p), int(nbytes),
                               int(reps), g))
    return {"h2d": g[0], "d2h": g[1], "both_h2d": g[2], "both_d2h": g[3], "both_sustained": g[4]}


def stream_release() -> int:
    """Free the streamer's cached per-GPU resources (fft_stream_release)."""
    return int(_lib.fft_stream_release())


def _host_ptr(a):
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.is_cuda or not a.is_contiguous():
                raise ValueError("expected a contiguous CPU tensor")
            return a.data_ptr(), a.numel() * a.element_size()
    except ImportError:
        pass
    import numpy as np
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("expected a C-contiguous array")
        return a.ctypes.data, a.nbytes
    raise TypeError("expected a torch CPU tensor or numpy array")


def file_records(file_bytes: int, record_len: int) -> int:
    r = int(_lib.fft_file_records(int(file_bytes), int(record_len)))
    if r < 0:
        raise FFTError(-r, last_error())
    return r


def partition(total_records: int, nparts: int, part: int) -> tuple[int, int]:
    """(first, count) of part `part` of `nparts` contiguous record ranges."""
    f, c = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.fft_partition(int(total_records), int(nparts), int(part), ctypes.byref(f), ctypes.byref(c)))
    return f.value, c.value
