"""GPU parity on the path the benchmarks actually run: the default (AUTO)
plan at every pipelined size, with batches that wrap the plan's L2 ring at
least twice, and the full config-3 workload.

The pipelined four-step (`k_pipe2` / `k_pipe3`) keeps the
intermediate of record r in ring slot r mod S.  Only a batch larger than S
makes an A-task reuse a slot, i.e. exercises the write-after-read waits and
the `discard.global.L2` + rewrite of a slot; a batch of 2S + 3 records turns
the ring over twice plus a ragged tail.  Checks per (N, direction):

* every record is bit-identical to the same record transformed alone with a
  batch-1 plan (batch independence; reading c13) — this covers
  every record, including all of those written through reused slots;
* a seeded sample of >= 8 records, always including the first, the last and
  records r >= S (second and third generation of a slot), matches the CPU
  oracle within the north_star bar 1e-5 log2 N (reading c10).

Inputs are the seeded SplitMix64 stream generated on the GPU;
the oracle's inputs are regenerated from (seed, r) on the host by `synth`.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

bf = pytest.importorskip("paper_1407_6915_b200")
from synth import gpu as sg  # noqa: E402

PIPE_SIZES = [2 ** k for k in range(15, 23)]   # AUTO is single pass up to 2^14


def ring_slots(n):
    with bf.Plan(n, 1) as p:
        info = p.info()
    assert info["variant_name"] == "pipe", info
    return info["scratch_bytes"] // (8 * n), info


def sample_with_wrap(b, s, count=8, seed=synth.SAMPLE_SEED):
    """First, last, records in the second and third generation of their slot,
    and seeded picks."""
    idx = {0, b - 1, s, min(b - 1, s + 1), min(b - 1, 2 * s), min(b - 1, 2 * s + 1)}
    for r in synth.sample_indices(b, count, seed):
        if len(idx) >= count:
            break
        idx.add(int(r))
    return np.array(sorted(idx))


def transform(x, n, b, direction):
    y = torch.empty_like(x)
    with bf.Plan(n, b, direction) as p:
        p.exec(x, y)
    torch.cuda.synchronize()
    return y


@pytest.mark.parametrize("direction", [bf.FFT_FORWARD, bf.FFT_INVERSE])
@pytest.mark.parametrize("n", PIPE_SIZES)
def test_default_plan_wraps_ring(n, direction):
    s, info = ring_slots(n)
    b = 2 * s + 3
    seed = synth.DEFAULT_SEED + 17 * n + (direction > 0)
    x = torch.empty((b, n), dtype=torch.complex64, device="cuda")
    sg.fill_random(x, seed)
    y = transform(x, n, b, direction)
    # every record vs the same record alone (batch-1 plan: no slot is ever reused)
    y1 = torch.empty_like(x)
    with bf.Plan(n, 1, direction) as p1:
        for r in range(b):
            p1.exec(x[r:r + 1], y1[r:r + 1])
    torch.cuda.synchronize()
    diff = (y.view(torch.float32) != y1.view(torch.float32)).view(b, -1).any(dim=1)
    bad = torch.nonzero(diff).flatten().tolist()
    assert not bad, f"N={n} dir={direction} S={s}: records not bit-identical to batch-1: {bad[:10]}"
    # seeded sample (including reused slots) vs the oracle
    idx = sample_with_wrap(b, s)
    assert idx.max() >= s
    x_h = np.stack([synth.random_records(seed, n, int(r), 1)[0] for r in idx])
    assert np.array_equal(x[torch.from_numpy(idx).cuda()].cpu().numpy(), x_h)
    err = oracle.rel_l2(y[torch.from_numpy(idx).cuda()].cpu().numpy(), oracle.records_c64(x_h, direction))
    assert np.all(err <= oracle.tolerance(n)), (n, direction, s, idx[err.argmax()], err.max())
    del x, y, y1
    torch.cuda.empty_cache()


def test_full_config3_sampled():
    # BASELINE.json configs[2]: 2048 records of 2^20 points (16 GiB) in HBM, the
    # launch configuration `bench.py --config 3` times (one plan over the batch).
    n, b = 1 << 20, 2048
    s, info = ring_slots(n)
    assert b > 2 * s
    seed = synth.DEFAULT_SEED
    x = torch.empty((b, n), dtype=torch.complex64, device="cuda")
    sg.fill_random(x, seed)
    y = transform(x, n, b, bf.FFT_FORWARD)
    idx = sample_with_wrap(b, s, count=8)
    x_h = np.stack([synth.random_records(seed, n, int(r), 1)[0] for r in idx])
    ti = torch.from_numpy(idx).cuda()
    assert np.array_equal(x[ti].cpu().numpy(), x_h)
    y_s = y[ti].cpu().numpy()
    err = oracle.rel_l2(y_s, oracle.records_c64(x_h, oracle.FORWARD))
    assert np.all(err <= oracle.tolerance(n)), (idx[err.argmax()], err.max())
    # the same records alone are bit-identical
    with bf.Plan(n, 1) as p1:
        for j, r in enumerate(idx):
            o = torch.empty((1, n), dtype=torch.complex64, device="cuda")
            p1.exec(x[int(r):int(r) + 1], o)
            torch.cuda.synchronize()
            assert np.array_equal(o.cpu().numpy()[0], y_s[j]), int(r)
    del x, y
    torch.cuda.empty_cache()
