"""Seeded synthetic signal generator shared by the oracle side and the GPU side.

Holds none of the method's arithmetic (no transform, no twiddle): only the
counter-based random numbers and structured test signals that feed both.
Recipe:

* canonical SplitMix64 in counter mode:
  ``out(seed, i) = mix(seed + (i + 1) * 0x9E3779B97F4A7C15)``;
* ``f(h) = (h >> 40) * 2^-23 - 1`` — uniform on [-1, 1), exact in fp32;
* global complex sample ``s`` (= record * N + index) has
  ``re = f(out(seed, 2 s))`` and ``im = f(out(seed, 2 s + 1))``.

So any record of any shard or file can be regenerated independently on any
host.  ``synth/csrc/synth_fill.cu`` implements the same generator as a CUDA
fill kernel (bit-identical, checked by a GPU test) so multi-GiB benchmark
inputs are created in HBM without a host round trip.

Structured records (SPEC.md:463-469 ``gen`` kinds): impulse, constant, real
tone ``cos(2 pi k0 j / N)`` and complex tone ``exp(+2 pi i k0 j / N)``,
computed in double and rounded once to fp32.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
DEFAULT_SEED = 0x14076915
SAMPLE_SEED = 0x5EED
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def splitmix64(seed: int, idx) -> np.ndarray:
    """out(seed, i) for an array of counters i (uint64 arithmetic mod 2^64)."""
    i = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(np.uint64(seed) + (i + np.uint64(1)) * GOLDEN)


def unit_float(h: np.ndarray) -> np.ndarray:
    """f(h) = (h >> 40) * 2^-23 - 1, exactly representable in fp32."""
    return ((h >> np.uint64(40)).astype(np.float64) * 2.0 ** -23 - 1.0).astype(np.float32)


def random_samples(seed: int, first: int, count: int) -> np.ndarray:
    """Global complex samples [first, first + count) as complex64."""
    s = np.arange(first, first + count, dtype=np.uint64)
    out = np.empty(count, dtype=np.complex64)
    v = out.view(np.float32)
    v[0::2] = unit_float(splitmix64(seed, np.uint64(2) * s))
    v[1::2] = unit_float(splitmix64(seed, np.uint64(2) * s + np.uint64(1)))
    return out


def random_records(seed: int, n: int, first_record: int, count: int) -> np.ndarray:
    """Records [first_record, first_record + count) of length n, shape [count, n]."""
    return random_samples(seed, first_record * n, count * n).reshape(count, n)


def record(kind: str, n: int, r: int = 0, seed: int = DEFAULT_SEED) -> np.ndarray:
    """One structured record of length n (complex64).

    kinds: ``random`` (record r of the seeded stream), ``impulse`` (delta at
    0), ``constant`` (all ones), ``tone`` (real cosine at bin r mod n),
    ``ctone`` (complex exponential at bin r mod n), ``zeros``.
    """
    j = np.arange(n, dtype=np.float64)
    k0 = r % n
    if kind == "random":
        return random_records(seed, n, r, 1)[0]
    if kind == "impulse":
        x = np.zeros(n, np.complex64)
        x[0] = 1
        return x
    if kind == "constant":
        return np.ones(n, np.complex64)
    if kind == "zeros":
        return np.zeros(n, np.complex64)
    if kind == "tone":
        return np.cos(2.0 * np.pi * ((k0 * j) % n) / n).astype(np.complex64)
    if kind == "ctone":
        return np.exp(2j * np.pi * ((k0 * j) % n) / n).astype(np.complex64)
    raise ValueError(f"unknown record kind {kind!r}")


def sample_indices(total: int, count: int, seed: int = SAMPLE_SEED) -> np.ndarray:
    """Sorted distinct record indices for sampled parity: always the first and
    last record plus seeded picks in between."""
    if total <= count:
        return np.arange(total)
    picks = {0, total - 1}
    i = 0
    while len(picks) < count:
        picks.add(int(splitmix64(seed, i) % np.uint64(total)))
        i += 1
    return np.array(sorted(picks), dtype=np.int64)
