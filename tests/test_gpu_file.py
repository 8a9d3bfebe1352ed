"""GPU tests of the file pipeline (fft_file: partition -> stream -> write by
offset) and the host streamer (fft_exec_host) against the oracle, plus the
identity-kernel byte-exact round trip and the
SPEC error conventions."""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
bf = pytest.importorskip("paper_1407_6915_b200")


def write_file(path, samples):
    np.asarray(samples, dtype="<c8").tofile(path)
    return os.path.getsize(path)


def read_c64(path, n):
    return np.fromfile(path, dtype="<c8").reshape(-1, n)


def test_config1_file_forward(tmp_path):
    # BASELINE.json configs[0]: 16 records x 1024-point complex64 forward FFT
    # from a synthetic seeded file.
    n, r = 1024, 16
    src, dst = tmp_path / "in.c64", tmp_path / "out.c64"
    write_file(src, synth.random_samples(synth.DEFAULT_SEED, 0, n * r))
    st = bf.fft_file(str(src), str(dst), n, 1)
    assert st["records"] == r and st["bytes_in"] == r * 8 * n
    y = read_c64(dst, n)
    ref = oracle.file_transform(src.read_bytes(), n)
    assert np.all(oracle.rel_l2(y, ref) <= oracle.tolerance(n))
    assert not os.path.exists(str(dst) + ".tmp")


def test_tail_padding_and_output_size(tmp_path):
    n = 1024
    s = synth.random_samples(3, 0, 5 * n + 100)
    src, dst = tmp_path / "in.c64", tmp_path / "out.c64"
    write_file(src, s)
    bf.fft_file(str(src), str(dst), n, 1)
    assert os.path.getsize(dst) == 6 * 8 * n           # R*8N, final record zero-padded
    y = read_c64(dst, n)
    ref = oracle.file_transform(src.read_bytes(), n)
    assert np.all(oracle.rel_l2(y, ref) <= oracle.tolerance(n))


@pytest.mark.parametrize("n", [256, 1 << 16])
def test_identity_byte_exact(tmp_path, n):
    src, dst = tmp_path / "in.c64", tmp_path / "out.c64"
    write_file(src, synth.random_samples(11, 0, 37 * n))
    bf.fft_file(str(src), str(dst), n, 1, direction=bf.FFT_IDENTITY, chunk_bytes=8 * n * 5)
    assert src.read_bytes() == dst.read_bytes()


@pytest.mark.parametrize("n,variant", [(1024, 0), (1 << 16, 0), (1 << 18, 0), (1 << 16, 3)])
def test_chunking_and_streaming_bit_identical_to_in_hbm(tmp_path, n, variant):
    # results depend only on (N, dir): not on chunk size, GPU count or path
    r = 23
    s = synth.random_samples(21, 0, r * n)
    src = tmp_path / "in.c64"
    write_file(src, s)
    outs = []
    for cb in (8 * n * 4, 8 * n * 7, 0):
        dst = tmp_path / f"out_{cb}.c64"
        bf.fft_file(str(src), str(dst), n, 1, chunk_bytes=cb, variant=variant)
        outs.append(read_c64(dst, n))
    x = torch.from_numpy(s.reshape(r, n)).cuda()
    y = torch.empty_like(x)
    with bf.Plan(n, r, bf.FFT_FORWARD, variant) as p:
        p.exec(x, y)
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    for o in outs:
        assert np.array_equal(o, y)
    ng = torch.cuda.device_count()
    if ng > 1:
        dst = tmp_path / "out_multi.c64"
        bf.fft_file(str(src), str(dst), n, ng, chunk_bytes=8 * n * 3, variant=variant)
        assert np.array_equal(read_c64(dst, n), y)


def test_forward_then_inverse_pipeline(tmp_path):
    # forward pipeline then inverse pipeline -> <= 1e-5 vs original
    n = 4096
    s = synth.random_samples(8, 0, 9 * n)
    a, b, c = tmp_path / "a", tmp_path / "b", tmp_path / "c"
    write_file(a, s)
    bf.fft_file(str(a), str(b), n, 1, direction=bf.FFT_FORWARD)
    bf.fft_file(str(b), str(c), n, 1, direction=bf.FFT_INVERSE)
    e = oracle.rel_l2(read_c64(c, n), s.reshape(-1, n))
    assert np.all(e <= 1e-5)


def test_sine3_spectral_check(tmp_path):
    # SPEC.md:469 / :515: sine:3 records -> peaks at bins 3 and N-3 of N/2 +- 1%,
    # off-peak energy < 1% of total, for every record.
    n, r = 1024, 8
    rec = synth.record("tone", n, 3)
    src, dst = tmp_path / "in", tmp_path / "out"
    write_file(src, np.tile(rec, r))
    bf.fft_file(str(src), str(dst), n, 1)
    mag = np.abs(read_c64(dst, n))
    assert np.all(np.abs(mag[:, [3, n - 3]] - n / 2) <= 0.01 * n / 2)
    off = np.delete(mag, [3, n - 3], axis=1)
    assert np.all((off ** 2).sum(1) < 0.01 * (mag ** 2).sum(1))


@pytest.mark.parametrize("pinned", [True, False])
def test_exec_host_matches_device(pinned):
    n, r = 1 << 16, 37
    s = torch.from_numpy(synth.random_records(4, n, 0, r))
    h = s.pin_memory() if pinned else s.clone()
    out = torch.empty_like(h).pin_memory() if pinned else torch.empty_like(h)
    st = bf.exec_host(h, n, bf.FFT_FORWARD, 0, out=out, chunk_bytes=8 * n * 8)
    assert st["records"] == r and st["chunks"] == 5
    x = s.cuda()
    with bf.Plan(n, r) as p:
        y = p.exec(x, torch.empty_like(x))
    torch.cuda.synchronize()
    assert torch.equal(out, y.cpu())
    assert torch.equal(h, s)      # out-of-place: input untouched


def test_file_errors(tmp_path):
    out = tmp_path / "out"
    with pytest.raises(bf.FFTError) as ei:
        bf.fft_file(str(tmp_path / "missing"), str(out), 1024, 1)
    assert ei.value.code == 8
    bad = tmp_path / "bad"
    bad.write_bytes(b"\0" * 12)
    with pytest.raises(bf.FFTError) as ei:
        bf.fft_file(str(bad), str(out), 1024, 1)
    assert ei.value.code == 4
    empty = tmp_path / "empty"
    empty.write_bytes(b"")
    with pytest.raises(bf.FFTError) as ei:
        bf.fft_file(str(empty), str(out), 1024, 1)
    assert ei.value.code == 9
    good = tmp_path / "good"
    write_file(good, np.zeros(2048, np.complex64))
    with pytest.raises(bf.FFTError) as ei:
        bf.fft_file(str(good), str(out), 1024, 99)
    assert ei.value.code == 5
    assert not out.exists() and not os.path.exists(str(out) + ".tmp")


def test_stream_cache_and_release(tmp_path):
    # repeated streamed calls reuse cached per-GPU resources; release frees them
    n = 4096
    s = torch.from_numpy(synth.random_records(6, n, 0, 40)).pin_memory()
    out1 = torch.empty_like(s).pin_memory()
    out2 = torch.empty_like(s).pin_memory()
    bf.exec_host(s, n, bf.FFT_FORWARD, 0, out=out1, chunk_bytes=8 * n * 16)
    bf.exec_host(s, n, bf.FFT_FORWARD, 0, out=out2, chunk_bytes=8 * n * 16)
    assert torch.equal(out1, out2)
    assert bf.stream_release() >= 1
    bf.exec_host(s, n, bf.FFT_FORWARD, 0, out=out2, chunk_bytes=8 * n * 16)
    assert torch.equal(out1, out2)


@pytest.mark.parametrize("n", [1 << 13, 1 << 16])
def test_file_inverse_roundtrip_pipelined(tmp_path, n):
    # the default (pipelined four-step) variant through the file pipeline, both directions
    s = synth.random_samples(12, 0, 19 * n)
    a, b, c = tmp_path / "a", tmp_path / "b", tmp_path / "c"
    write_file(a, s)
    bf.fft_file(str(a), str(b), n, 1, direction=bf.FFT_FORWARD, chunk_bytes=8 * n * 6)
    ref = oracle.file_transform(a.read_bytes(), n)
    assert np.all(oracle.rel_l2(read_c64(b, n), ref) <= oracle.tolerance(n))
    bf.fft_file(str(b), str(c), n, 1, direction=bf.FFT_INVERSE, chunk_bytes=8 * n * 5)
    assert np.all(oracle.rel_l2(read_c64(c, n), s.reshape(-1, n)) <= 2 * oracle.tolerance(n))


def test_file_range_pieces_equal_whole_file(tmp_path):
    # fft_file_range (one GPU's / node's share): ranges written into one
    # pre-sized output reproduce fft_file bit for bit; a ragged tail record included
    n = 4096
    s = synth.random_samples(31, 0, 29 * n + 77)
    src, whole, parts = tmp_path / "in", tmp_path / "whole", tmp_path / "parts"
    write_file(src, s)
    bf.fft_file(str(src), str(whole), n, 1)
    r = bf.file_records(os.path.getsize(src), n)
    with open(parts, "wb") as f:
        f.truncate(r * 8 * n)
    for g in (2, 0, 1):                        # any order: writes are positional
        first, count = bf.partition(r, 3, g)
        st = bf.file_range(str(src), str(parts), n, first, count, device=0,
                           options=bf.StreamOptions(chunk_bytes=8 * n * 4))
        assert st["records"] == count
    assert whole.read_bytes() == parts.read_bytes()
    with pytest.raises(bf.FFTError) as ei:
        bf.file_range(str(src), str(parts), n, r - 1, 2)
    assert ei.value.code == 4


@pytest.mark.parametrize("pinned", [True, False])
def test_stream_host_ring_taps(pinned):
    # fft_stream_host: a logical stream longer than its input ring (record r reads
    # ring record r mod K); taps capture sampled outputs along the whole stream.
    n, k, total = 1024, 48, 1000
    ring = torch.from_numpy(synth.random_records(41, n, 0, k))
    ring = ring.pin_memory() if pinned else ring.clone()
    out = torch.empty((64, n), dtype=torch.complex64)
    out = out.pin_memory() if pinned else out
    taps = [0, 1, 47, 48, 100, 511, 998, 999]
    o = bf.StreamOptions(n=n, chunk_bytes=8 * n * 16, taps=taps, timeline=100)
    st = bf.stream_host(ring, out, n, total, options=o)
    assert st["records"] == total and st["taps"] == len(taps) and st["chunks"] == 63
    x = ring.cuda()
    with bf.Plan(n, k) as p:
        y = p.exec(x, torch.empty_like(x)).cpu().numpy()
    torch.cuda.synchronize()
    for j, r in enumerate(taps):               # bit-identical to the in-HBM transform
        assert np.array_equal(o.tap_out[j], y[r % k]), r
    assert np.all(oracle.rel_l2(o.tap_out, oracle.records_c64(ring.numpy()[np.array(taps) % k], -1))
                  <= oracle.tolerance(n))
    # the output ring holds the last records: record r at out[r % 64]
    for r in range(total - 64, total):
        assert np.array_equal(out.numpy()[r % 64], y[r % k])
    tl = o.timeline_out[:st["chunks"]]
    assert np.all(np.isfinite(tl))
    if pinned:                                 # pinned ring: copied directly, no read stage
        assert np.all(tl[:, :2] == 0)
    assert np.all(tl[:, 3] >= tl[:, 2]) and np.all(tl[:, 4] >= tl[:, 3]) and np.all(tl[:, 5] >= tl[:, 4])


def test_stream_overlap_timeline():
    # copies overlap compute in both directions: with D chunks in flight, chunk k+1's
    # H2D starts before chunk k's D2H ends
    n, k = 1 << 16, 64
    ring = torch.from_numpy(synth.random_records(5, n, 0, k)).pin_memory()
    out = torch.empty_like(ring).pin_memory()
    o = bf.StreamOptions(n=n, chunk_bytes=8 * n * 8, timeline=64)
    st = bf.stream_host(ring, out, n, 8 * k, options=o)
    tl = o.timeline_out[:st["chunks"]]
    overlapped = np.sum(tl[1:, 2] < tl[:-1, 5])
    assert overlapped >= len(tl) // 2, tl[:6]


@pytest.mark.parametrize("direct", [False, True])
def test_file_direct_io_option(tmp_path, direct):
    # O_DIRECT where the file system supports it (else buffered, reported in stats)
    n = 1024
    s = synth.random_samples(13, 0, 40 * n + 8)
    src, dst = tmp_path / "in", tmp_path / "out"
    write_file(src, s)
    st = bf.fft_file(str(src), str(dst), n, 1, options=bf.StreamOptions(chunk_bytes=8 * n * 7, direct_io=direct))
    if not direct:
        assert st["direct_io"] == 0
    ref = oracle.file_transform(src.read_bytes(), n)
    assert np.all(oracle.rel_l2(read_c64(dst, n), ref) <= oracle.tolerance(n))
    assert os.path.getsize(dst) == 41 * 8 * n


def test_numa_node_query():
    node = bf.numa_node(0)
    assert isinstance(node, int) and node >= -1
