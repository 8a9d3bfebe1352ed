"""Pins for the CPU oracle (oracle/): closed forms, the paper/SPEC worked
examples, brute force, invariants and an independent library cross-check.

Nothing here compares the oracle with itself: every expected value comes from
a closed form, a golden fixture with its citation, a mathematical identity, or
numpy.fft (pocketfft — a library the oracle does not use).  The two oracle
algorithms (direct DFT, recursive radix-2) are independent code paths; the
brute-force test compares them only after both are pinned to closed forms.
"""
import numpy as np
import pytest

import oracle
import synth
from conftest import parse_cvec, read_golden

POW2 = [2 ** k for k in range(1, 13)]


def rnd(n, seed=1, count=1):
    return synth.random_records(seed, n, 0, count).astype(np.complex128)


@pytest.mark.parametrize("row", read_golden("spec_fft_examples.txt"), ids=lambda r: r[0])
@pytest.mark.parametrize("fn", ["dft", "fft"])
def test_spec_worked_examples(row, fn):
    name, n, d, x, y, _cite = row
    x, y = parse_cvec(x), parse_cvec(y)
    assert x.size == int(n)
    out = getattr(oracle, fn)(x, int(d))
    np.testing.assert_allclose(out, y, rtol=0, atol=1e-14)


def test_n4_forward_twiddles_spec49():
    # SPEC.md:49 plan_create(4,1,forward) -> twiddle_table = [1+0i, 0-1i]:
    # the spectrum of the shifted impulse is W_4^k, its bins 0,1 are that table.
    for fn in (oracle.dft, oracle.fft):
        out = fn(np.array([0, 1, 0, 0], np.complex128))
        np.testing.assert_allclose(out[:2], [1 + 0j, -1j], atol=1e-15)


@pytest.mark.parametrize("n", POW2)
@pytest.mark.parametrize("fn", ["dft", "fft"])
def test_closed_forms(n, fn):
    f = getattr(oracle, fn)
    if fn == "dft" and n > 1024:
        pytest.skip("direct DFT closed forms checked up to 1024")
    tol = 1e-12 * n
    # impulse -> all ones
    x = np.zeros(n, np.complex128); x[0] = 1
    np.testing.assert_allclose(f(x), np.ones(n), atol=tol)
    # constant -> N * delta
    e = np.zeros(n, np.complex128); e[0] = n
    np.testing.assert_allclose(f(np.ones(n, np.complex128)), e, atol=tol)
    # shifted impulse delta[j-s] -> exp(-2 pi i s k / N)
    s = (3 * n) // 4 if n >= 4 else 1
    x = np.zeros(n, np.complex128); x[s] = 1
    k = np.arange(n)
    np.testing.assert_allclose(f(x), np.exp(-2j * np.pi * ((s * k) % n) / n), atol=tol)
    # complex tone exp(+2 pi i k0 j / N) -> N * delta[k - k0]
    k0 = (5 * n) // 8 % n
    j = np.arange(n)
    x = np.exp(2j * np.pi * ((k0 * j) % n) / n)
    e = np.zeros(n, np.complex128); e[k0] = n
    np.testing.assert_allclose(f(x), e, atol=tol)
    # real tone cos(2 pi k0 j / N) -> N/2 at k0 and N-k0
    if n >= 4:
        k0 = 1 + n // 8
        x = np.cos(2 * np.pi * ((k0 * j) % n) / n).astype(np.complex128)
        e = np.zeros(n, np.complex128); e[k0] = n / 2; e[n - k0] = n / 2
        np.testing.assert_allclose(f(x), e, atol=tol)


@pytest.mark.parametrize("fn", ["dft", "fft"])
def test_inverse_closed_forms(fn):
    f = getattr(oracle, fn)
    for n in (2, 8, 64, 512):
        # inverse of N*delta[k-k0] is exp(+2 pi i k0 j/N) (SPEC.md:90 scaling 1/N)
        k0 = n // 2 - 1 if n > 2 else 1
        X = np.zeros(n, np.complex128); X[k0] = n
        j = np.arange(n)
        np.testing.assert_allclose(f(X, oracle.INVERSE),
                                   np.exp(2j * np.pi * ((k0 * j) % n) / n), atol=1e-12 * n)


def test_spec_sine3_golden():
    (row,) = read_golden("spec_sine3.txt")
    n, k0 = int(row[0]), int(row[1])
    bins = [int(b) for b in row[2].split(",")]
    peak, tol = float(row[3]), float(row[4])
    x = synth.record("tone", n, k0)
    for fn in (oracle.dft, oracle.fft):
        mag = np.abs(fn(x.astype(np.complex128)))
        np.testing.assert_allclose(mag[bins], peak, rtol=1e-6)
        off = np.delete(mag, bins)
        assert off.max() < tol
        assert np.sum(off ** 2) < 0.01 * np.sum(mag ** 2)


def test_non_power_of_two_dft_defined():
    # "any length-6 input -> defined (oracle supports non-power-of-two)".
    n = 6
    j = np.arange(n)
    for k0 in range(n):
        x = np.exp(2j * np.pi * k0 * j / n)
        e = np.zeros(n, np.complex128); e[k0] = n
        np.testing.assert_allclose(oracle.dft(x), e, atol=1e-13)
    with pytest.raises(ValueError):
        oracle.fft(np.ones(6))           # radix-2 needs a power of two
    with pytest.raises(ValueError):
        oracle.fft(np.ones(4), 2)        # direction must be -1 or +1


@pytest.mark.parametrize("n", [2 ** k for k in range(0, 7)])
def test_bruteforce_fft_vs_dft_small(n):
    # north_star: "checked ... against the brute-force DFT on N <= 64"
    x = rnd(n, seed=7 + n, count=4)
    for d in (oracle.FORWARD, oracle.INVERSE):
        for r in x:
            a, b = oracle.fft(r, d), oracle.dft(r, d)
            assert oracle.rel_l2(a, b)[0] <= 1e-13


@pytest.mark.parametrize("n", [256, 1024, 4096])
def test_bruteforce_fft_vs_dft_medium(n):
    r = rnd(n, seed=99)[0]
    assert oracle.rel_l2(oracle.fft(r), oracle.dft(r))[0] <= 1e-12


@pytest.mark.parametrize("k", list(range(1, 23)))
def test_numpy_crosscheck(k):
    # Independent library routine (pocketfft, double) — never used by the oracle.
    n = 2 ** k
    x = rnd(n, seed=k)[0]
    ref_f = np.fft.fft(x)
    assert oracle.rel_l2(oracle.fft(x), ref_f)[0] <= 1e-12
    if k <= 14:
        assert oracle.rel_l2(oracle.fft(x, oracle.INVERSE), np.fft.ifft(x))[0] <= 1e-12


@pytest.mark.parametrize("n", [2, 16, 1024, 65536])
def test_invariants(n):
    x, y = rnd(n, seed=3, count=2)
    X, Y = oracle.fft(x), oracle.fft(y)
    # Parseval: sum|x|^2 = (1/N) sum|X|^2
    assert abs(np.sum(np.abs(x) ** 2) - np.sum(np.abs(X) ** 2) / n) <= 1e-12 * np.sum(np.abs(x) ** 2)
    # linearity
    a, b = 0.75 - 0.5j, -1.25 + 2j
    assert oracle.rel_l2(oracle.fft(a * x + b * y), a * X + b * Y)[0] <= 1e-13
    # round trip
    assert oracle.rel_l2(oracle.fft(X, oracle.INVERSE), x)[0] <= 1e-13
    # real input -> Hermitian spectrum X[N-k] = conj(X[k])
    R = oracle.fft(x.real.astype(np.complex128))
    k = np.arange(1, n)
    np.testing.assert_allclose(R[n - k], np.conj(R[k]), atol=1e-12 * n)
    # shift theorem fft(roll(x, s))[k] = W^{s k} X[k]
    s = n // 3 + 1
    kk = np.arange(n)
    np.testing.assert_allclose(oracle.fft(np.roll(x, s)),
                               np.exp(-2j * np.pi * ((s * kk) % n) / n) * X,
                               atol=1e-11 * np.sqrt(n))


def test_batch_records_independent_and_exact_promotion():
    n, b = 256, 9
    x64 = synth.random_records(11, n, 0, b)
    out = oracle.records_c64(x64, oracle.FORWARD, threads=2)
    for r in range(b):
        one = oracle.fft(x64[r].astype(np.complex128))
        assert np.array_equal(out[r], one)           # bit-identical per record
    out_d = oracle.records_c64(x64[:3], oracle.FORWARD, algo="dft")
    assert np.all(oracle.rel_l2(out[:3], out_d) <= 1e-12)


def test_file_transform_tail_padding():
    # reading c6: final record zero-padded; SPEC.md:149/158 padding semantics.
    n = 64
    s = synth.random_samples(5, 0, 3 * n + 17)
    raw = s.astype("<c8").tobytes()
    out = oracle.file_transform(raw, n)
    assert out.shape == (4, n)
    last = np.zeros(n, np.complex64); last[:17] = s[3 * n:]
    assert np.array_equal(out[3], oracle.fft(last.astype(np.complex128)))
    assert np.array_equal(out[1], oracle.fft(s[n:2 * n].astype(np.complex128)))
    with pytest.raises(ValueError):
        oracle.file_transform(raw[:-3], n)            # not a multiple of 8 bytes
    with pytest.raises(ValueError):
        oracle.file_transform(b"", n)                 # empty input


def test_rel_l2_semantics():
    ref = np.array([[1, 0], [0, 0]], np.complex128)
    y = np.array([[1, 1e-3], [0, 0]], np.complex128)
    e = oracle.rel_l2(y, ref)
    assert e[0] == pytest.approx(1e-3) and e[1] == 0.0
    assert oracle.rel_l2(np.array([1e-30 + 0j]), np.array([0j]))[0] == np.inf
    assert oracle.tolerance(1024) == pytest.approx(1e-4)
