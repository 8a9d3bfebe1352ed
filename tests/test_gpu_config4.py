"""Config 4 at full size (BASELINE.json configs[3]): a 1 TiB
logical signal of 1024-point complex64 records (2^27 records, the paper's
record length) streamed host -> GPU -> host through
fft_stream_host on one GPU — the launch configuration tools/stream_tib.py
times — with one tapped record per GiB of the stream (1024 taps, SURVEY's
">= 1 sampled record per GiB") checked against the CPU oracle within the
north_star bar, and bit for bit against the in-HBM transform of the same
input (reading c13: the streamed result equals the in-HBM one).

Source: a 1 GiB pinned capture ring of seeded records replayed (record r
reads ring record r mod K; "host-memory source/sink, disk excluded"); sink: a
rolling pinned ring.  Inputs are regenerated for the oracle from (seed, r mod K)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
bf = pytest.importorskip("paper_1407_6915_b200")


def test_one_tib_logical_stream_tapped_parity():
    n = 1024
    rb = 8 * n
    total = (1 << 40) // rb                 # 134,217,728 records (P:49 arithmetic, reading c12)
    k = (1 << 30) // rb                     # 1 GiB capture ring
    seed = synth.DEFAULT_SEED
    ring = bf.HostBuffer(k, n, 0)
    out = bf.HostBuffer(k, n, 0)
    x_h = synth.random_records(seed, n, 0, k)
    ring.a[:] = x_h
    taps = np.arange(0, total, (1 << 30) // rb, dtype=np.int64)       # one per GiB
    taps[1:] += synth.sample_indices(k, len(taps) - 1)[: len(taps) - 1] % k  # spread inside each GiB
    taps = np.unique(taps)
    o = bf.StreamOptions(n=n, chunk_bytes=256 << 20, taps=taps)
    st = bf.stream_host(ring.a, out.a, n, total, options=o)
    assert st["records"] == total and st["taps"] == len(taps) >= 1024
    rid = taps % k
    ref = oracle.records_c64(x_h[rid], oracle.FORWARD)
    err = oracle.rel_l2(o.tap_out, ref)
    assert np.all(err <= oracle.tolerance(n)), (taps[err.argmax()], err.max())
    x = torch.from_numpy(x_h[np.unique(rid)]).cuda()
    with bf.Plan(n, x.shape[0]) as p:
        y = p.exec(x, torch.empty_like(x)).cpu().numpy()
    pos = {r: i for i, r in enumerate(np.unique(rid))}
    for j, r in enumerate(rid):
        assert np.array_equal(o.tap_out[j], y[pos[r]]), taps[j]
    ring.close()
    out.close()
