"""Interleaving stress of the pipelined four-step's cross-CTA protocol
(the race check compute-sanitizer would give is closed on this
pool: profiles/r02_compute_sanitizer_closed.txt).

libblockfft_stress.so is the product library with the pipelined kernels
compiled with -DBFFT_STRESS: pseudo-random sleeps of up to ~2 us at every
synchronisation point of the task graph (producer before its dependency
waits and stage refills, release warps before publishing, compute warps
before reading a stage and before writing the ring, k_pipe's A/B tasks).
The arithmetic is identical, so any result that is not bit-identical to the
product build's exposes a missing wait or an unordered publication: a B-task
reading a slot before every A-task wrote it, an A-task overwriting a slot a
B-task still reads, a stage refilled while still in use.  Every case wraps
the L2 ring (default ring size, or the ring forced to LAG + 1 slots), runs
three times, both directions where listed."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
bf = pytest.importorskip("paper_1407_6915_b200")
from paper_1407_6915_b200 import _abi  # noqa: E402
from synth import gpu as sg  # noqa: E402

_stress = None


def stress_lib():
    global _stress
    if _stress is None:
        _stress = _abi.load(_abi.STRESS_LIB_PATH)
    return _stress


def run(lib, n, b, direction, x, y, **o):
    opts = _abi.PlanOpts(bf.VARIANT_PIPE, o.get("impl", 0), o.get("config", 0), 0, o.get("ring_records", 0),
                         o.get("ring_lag", 0))
    h = lib.fft_plan_create_opts(n, b, direction, ctypes.byref(opts))
    assert h, lib.fft_last_error()
    info = _abi.PlanInfo()
    assert lib.fft_plan_get_info(ctypes.c_void_p(h), ctypes.byref(info)) == 0
    rc = lib.fft_exec(ctypes.c_void_p(h), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    lib.fft_plan_destroy(ctypes.c_void_p(h))
    assert rc == 0, lib.fft_last_error()
    return info.ring_records


CASES = [
    # (n, batch or None = 2S+3 at the default ring, plan options, both directions)
    (1 << 14, None, {}, True),
    (1 << 16, 17, dict(ring_lag=3, ring_records=4), True),
    (1 << 16, 17, dict(impl=1, ring_lag=3, ring_records=4), False),
    (1 << 16, 17, dict(impl=2, config=1, ring_lag=3, ring_records=4), True),
    (1 << 18, 11, dict(impl=2, config=3, ring_lag=2, ring_records=3), False),
    (1 << 16, 17, dict(impl=3, ring_lag=3, ring_records=4), True),
    (1 << 16, 17, dict(impl=3, config=2, ring_lag=3, ring_records=4), False),
    (1 << 17, 11, dict(ring_lag=2, ring_records=3), False),
    (1 << 18, 11, dict(ring_lag=2, ring_records=3), False),
    (1 << 19, None, {}, False),
    (1 << 20, 9, dict(ring_lag=2, ring_records=3), True),
    (1 << 21, None, {}, False),
    (1 << 22, None, {}, True),
]


@pytest.mark.parametrize("n,b,o,both", CASES, ids=[f"2^{int(np.log2(c[0]))}-{i}" for i, c in enumerate(CASES)])
def test_stress_build_bit_identical(n, b, o, both):
    lib = stress_lib()
    if b is None:
        with bf.Plan(n, 1, bf.FFT_FORWARD, bf.VARIANT_PIPE, **o) as p:
            b = 2 * p.info()["ring_records"] + 3
    x = torch.empty((b, n), dtype=torch.complex64, device="cuda")
    sg.fill_random(x, 99 + n)
    for d in ((bf.FFT_FORWARD, bf.FFT_INVERSE) if both else (bf.FFT_FORWARD,)):
        ref = torch.empty_like(x)
        with bf.Plan(n, b, d, bf.VARIANT_PIPE, **o) as p:
            s_ring = p.info()["ring_records"]
            p.exec(x, ref)
        torch.cuda.synchronize()
        assert b > s_ring                                  # the ring wraps
        for rep in range(3):
            y = torch.full_like(x, float("nan"))
            assert run(lib, n, b, d, x, y, **o) == s_ring
            diff = (y.view(torch.float32) != ref.view(torch.float32)).view(b, -1).any(dim=1)
            bad = torch.nonzero(diff).flatten().tolist()
            assert not bad, f"N={n} dir={d} {o} rep {rep}: records differ under stress: {bad[:10]}"
    del x
    torch.cuda.empty_cache()
