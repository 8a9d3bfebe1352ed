"""GPU parity of overlapping records — the short-time Fourier transform
(fft_plan_create_stft, the paper's stated future work
PAPER.md:129) — against the CPU oracle: frame f is the n samples of the
signal starting at f*hop times the window (test-side framing, the plain
definition), each frame transformed by the oracle; relative L2 per frame
<= 1e-5 log2 n (reading c10).  Also: hop = n without a window is bit-identical
to the record transform; the file streamer (chunks re-read their n - hop halo)
is bit-identical to the in-HBM STFT across chunk sizes and GPU ranges."""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
bf = pytest.importorskip("paper_1407_6915_b200")


def frames_of(sig, n, hop, nframes, window=None):
    """Frame f = sig[f*hop : f*hop+n] (zero past the end) times the window."""
    out = np.zeros((nframes, n), np.complex64)
    for f in range(nframes):
        seg = sig[f * hop: f * hop + n]
        out[f, : seg.size] = seg
    if window is not None:
        out = (out * window.astype(np.float32)).astype(np.complex64)
    return out


def hann(n):
    return (0.5 - 0.5 * np.cos(2 * np.pi * np.arange(n) / n)).astype(np.float32)


@pytest.mark.parametrize("n,hop", [(256, 128), (1024, 256), (1024, 768), (1024, 1000), (4096, 1024),
                                   (8192, 4096), (8192, 4097), (1 << 14, 4096), (1 << 14, 4095), (1 << 16, 1 << 15),
                                   (1 << 16, 12345), (1024, 1500)])
@pytest.mark.parametrize("win", [False, True])
def test_stft_matches_oracle(n, hop, win):
    frames = max(3, min((1 << 21) // n, 257)) | 1
    length = (frames - 1) * hop + n
    sig = synth.random_samples(500 + n + hop, 0, length)
    w = hann(n) if win else None
    with bf.StftPlan(n, hop, frames, window=w) as p:
        info = p.info()
        y = p.exec(torch.from_numpy(sig).cuda())
    torch.cuda.synchronize()
    assert info["hop"] == hop
    # the window multiply rounds to fp32 exactly as the GPU does (x * w in fp32)
    ref = oracle.records_c64(frames_of(sig, n, hop, frames, w), oracle.FORWARD)
    err = oracle.rel_l2(y.cpu().numpy(), ref)
    assert np.all(err <= oracle.tolerance(n)), (n, hop, win, err.max())
    assert err.max() <= 2e-6


@pytest.mark.parametrize("n", [1024, 8192, 1 << 16])   # 8192: contiguous frames take k_rows_tma
def test_stft_hop_n_equals_records(n):
    b = 9
    sig = synth.random_samples(3, 0, b * n)
    x = torch.from_numpy(sig).cuda()
    with bf.StftPlan(n, n, b) as p:
        y1 = p.exec(x)
    with bf.Plan(n, b) as p:
        y2 = p.exec(x.view(b, n), torch.empty((b, n), dtype=torch.complex64, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)


@pytest.mark.parametrize("n,hop,fused", [(1 << 16, 1 << 15, True), (1 << 16, 12346, True), (1 << 16, 12345, False),
                                         (1 << 15, 1000, True), (1 << 15, 999, False), (1 << 15, 40000, True),
                                         (1 << 20, 1 << 19, True)])
def test_stft_long_frames_one_kernel(n, hop, fused):
    # frames longer than 2^14: an even hop is framed by k_pipe2's TMA tensor map
    # and windowed as its A-tiles are read (one kernel); an odd hop (TMA strides
    # are 16-byte multiples) goes through k_frames first.  Both vs the oracle.
    frames = 7
    length = (frames - 1) * hop + n
    sig = synth.random_samples(900 + hop, 0, length)
    w = hann(n)
    with bf.StftPlan(n, hop, frames, window=w) as p:
        info = p.info()
        y = p.exec(torch.from_numpy(sig).cuda())
    torch.cuda.synchronize()
    assert info["kernels_per_exec"] == (1 if fused else 2)
    ref = oracle.records_c64(frames_of(sig, n, hop, frames, w), oracle.FORWARD)
    err = oracle.rel_l2(y.cpu().numpy(), ref)
    assert np.all(err <= oracle.tolerance(n)), err.max()
    assert err.max() <= 2e-6, err.max()


def test_stft_errors():
    with pytest.raises(bf.FFTError) as ei:
        bf.StftPlan(1024, 0, 4)
    assert ei.value.code == 4
    with bf.StftPlan(1024, 512, 4) as p:
        with pytest.raises(ValueError):
            p.exec(torch.zeros(1024, dtype=torch.complex64, device="cuda"))   # too short
        x = torch.zeros(1024 * 4, dtype=torch.complex64, device="cuda")
        with pytest.raises(bf.FFTError) as ei:                                 # in/out overlap
            p.exec(x, x[: 4 * 1024].view(4, 1024))
        assert ei.value.code == 4


@pytest.mark.parametrize("n,hop", [(1024, 256), (4096, 3000), (1 << 16, 1 << 14)])
def test_stft_file_stream(tmp_path, n, hop):
    length = 37 * hop + n // 3                     # ragged end: the last frames are zero-padded
    sig = synth.random_samples(71, 0, length)
    w = hann(n)
    src = tmp_path / "sig.c64"
    sig.astype("<c8").tofile(src)
    nframes = 1 + -(-(length - n) // hop)
    outs = []
    for cb in (8 * n * 3, 8 * n * 7, 0):
        dst = tmp_path / f"stft_{cb}.c64"
        st = bf.fft_file(str(src), str(dst), n, 1, options=bf.StreamOptions(chunk_bytes=cb, hop=hop, window=w))
        assert st["records"] == nframes and os.path.getsize(dst) == nframes * 8 * n
        outs.append(np.fromfile(dst, "<c8").reshape(nframes, n))
    sig_pad = np.zeros((nframes - 1) * hop + n, np.complex64)
    sig_pad[:length] = sig
    with bf.StftPlan(n, hop, nframes, window=w) as p:
        yd = p.exec(torch.from_numpy(sig_pad).cuda()).cpu().numpy()
    for o in outs:
        assert np.array_equal(o, yd)               # chunking / halos do not change a bit
    ref = oracle.records_c64(frames_of(sig, n, hop, nframes, w), oracle.FORWARD)
    assert np.all(oracle.rel_l2(yd, ref) <= oracle.tolerance(n))
    # two GPU-sized ranges of frames through fft_file_range (each re-reads its halo)
    part = tmp_path / "parts.c64"
    with open(part, "wb") as f:
        f.truncate(nframes * 8 * n)
    for g in (1, 0):
        first, count = bf.partition(nframes, 2, g)
        bf.file_range(str(src), str(part), n, first, count, options=bf.StreamOptions(hop=hop, window=w))
    assert np.array_equal(np.fromfile(part, "<c8").reshape(nframes, n), yd)
