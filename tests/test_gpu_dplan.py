"""One transform larger than a GPU (fft_dplan_*): a
single record held as G contiguous slabs on G GPUs, transformed by the
distributed four-step whose transposes are peer stores over NVLink, against
the CPU oracle on the whole record (relative L2 <= 1e-5 log2 N, reading c10).
G = every visible GPU (1 on a one-GPU box: the same kernels, the peers being
the GPU itself) and G = 1; forward and inverse; natural order in and out."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
bf = pytest.importorskip("paper_1407_6915_b200")


def gpu_counts():
    n = torch.cuda.device_count()
    return sorted({1, n if n & (n - 1) == 0 else 1 << (n.bit_length() - 1)})


@pytest.mark.parametrize("g", gpu_counts())
@pytest.mark.parametrize("k", [12, 16, 21, 24])
@pytest.mark.parametrize("direction", [bf.FFT_FORWARD, bf.FFT_INVERSE])
def test_distributed_record_matches_oracle(g, k, direction):
    n = 1 << k
    x = synth.random_samples(900 + k, 0, n)
    per = n // g
    slabs = [torch.from_numpy(x[i * per:(i + 1) * per]).to(f"cuda:{i}") for i in range(g)]
    outs = [torch.empty_like(s) for s in slabs]
    with bf.DistPlan(n, g, direction) as p:
        n1, n2 = p.geometry()
        assert n1 * n2 == n and n1 % g == 0 and n2 % g == 0
        p.exec(slabs, outs)
    y = np.concatenate([o.cpu().numpy() for o in outs])
    ref = oracle.records_c64(x[None], direction)[0]
    err = oracle.rel_l2(y, ref)[0]
    assert err <= oracle.tolerance(n), (g, k, err)
    assert err <= 2e-6, err
    # inputs untouched out of place
    assert np.array_equal(np.concatenate([s.cpu().numpy() for s in slabs]), x)


def test_distributed_in_place_and_roundtrip():
    g = gpu_counts()[-1]
    n = 1 << 20
    x = synth.random_samples(5, 0, n)
    per = n // g
    slabs = [torch.from_numpy(x[i * per:(i + 1) * per]).to(f"cuda:{i}") for i in range(g)]
    with bf.DistPlan(n, g) as f, bf.DistPlan(n, g, bf.FFT_INVERSE) as b:
        f.exec(slabs)           # in place
        b.exec(slabs)
    z = np.concatenate([s.cpu().numpy() for s in slabs])
    assert oracle.rel_l2(z, x)[0] <= oracle.tolerance(n)


def test_distributed_plan_errors():
    with pytest.raises(bf.FFTError) as ei:
        bf.DistPlan(1000, 1)
    assert ei.value.code == 1
    with pytest.raises(bf.FFTError) as ei:
        bf.DistPlan(1 << 20, 3)
    assert ei.value.code == 5
    with pytest.raises(bf.FFTError) as ei:
        bf.DistPlan(1 << 20, 1, 0)
    assert ei.value.code == 3
