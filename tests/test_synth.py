"""Generator pins: canonical SplitMix64 known answers and fp32 exactness."""
import numpy as np

import synth
from conftest import read_golden


def test_splitmix64_known_answers():
    for seed, i, val in read_golden("splitmix64.txt"):
        assert int(synth.splitmix64(int(seed), int(i))) == int(val, 16)


def test_unit_float_exact_and_in_range():
    h = synth.splitmix64(synth.DEFAULT_SEED, np.arange(200000, dtype=np.uint64))
    f = synth.unit_float(h)
    assert f.dtype == np.float32
    assert f.min() >= -1.0 and f.max() < 1.0
    # exact: every value is a multiple of 2^-23 reproduced in float32
    q = (f.astype(np.float64) + 1.0) * 2 ** 23
    assert np.all(q == np.round(q))
    assert np.array_equal(q.astype(np.uint64), (h >> np.uint64(40)))
    assert abs(float(f.mean())) < 0.01


def test_record_addressing_is_global():
    n = 32
    a = synth.random_records(7, n, 3, 4)
    b = synth.random_samples(7, 3 * n, 4 * n).reshape(4, n)
    assert np.array_equal(a, b)
    assert np.array_equal(synth.record("random", n, 5, seed=7), a[2])
    assert not np.array_equal(synth.random_records(8, n, 3, 1), a[:1])


def test_structured_records():
    n = 16
    assert synth.record("impulse", n)[0] == 1 and np.count_nonzero(synth.record("impulse", n)) == 1
    assert np.all(synth.record("constant", n) == 1)
    t = synth.record("tone", n, 3)
    assert t.dtype == np.complex64 and np.all(t.imag == 0)
    assert abs(t[0] - 1) == 0


def test_sample_indices():
    idx = synth.sample_indices(1000, 16)
    assert idx[0] == 0 and idx[-1] == 999 and len(set(idx.tolist())) == 16
    assert np.all(np.diff(idx) > 0)
    assert np.array_equal(synth.sample_indices(5, 16), np.arange(5))
