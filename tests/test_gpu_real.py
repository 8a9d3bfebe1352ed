"""GPU parity of real-record transforms (fft_plan_create_real; SURVEY.md §8(f)
NEXT-1 — the paper's literal record, 1024 float32 samples = 4096 bytes,
PAPER.md:49) against the CPU oracle: the real record is promoted exactly to
complex and transformed by the oracle; the packed half spectrum the GPU
returns (out[0] = (X[0], X[n/2]), out[k] = X[k] for 0 < k < n/2) must match
those oracle bins within the north_star bar, relative L2 per record
<= 1e-5 log2 n.  The inverse is checked against the oracle inverse of the
Hermitian-extended spectrum (the plain definition of C2R).  Sizes 2^2..2^23,
ragged batches, in place and out of place, file and host-memory streaming."""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
bf = pytest.importorskip("paper_1407_6915_b200")


def real_records(seed, n, b):
    # seeded reals in [-1, 1): the SplitMix64 stream's samples, both parts used
    return synth.random_samples(seed, 0, b * n // 2).view(np.float32).reshape(b, n).copy()


def packed_from_full(X):
    """The packed half spectrum of full spectra X [B, n] (test-side bookkeeping)."""
    n = X.shape[1]
    P = X[:, : n // 2].copy()
    P[:, 0] = X[:, 0].real + 1j * X[:, n // 2].real
    return P


def full_from_packed(P):
    """Hermitian extension of packed half spectra [B, n/2] to full spectra [B, n]."""
    b, h = P.shape
    n = 2 * h
    X = np.zeros((b, n), np.complex128)
    X[:, 0] = P[:, 0].real
    X[:, h] = P[:, 0].imag
    X[:, 1:h] = P[:, 1:]
    X[:, h + 1:] = np.conj(P[:, 1:][:, ::-1])
    return X


def batch_for(n):
    return max(3, min((1 << 20) // n, 257)) | 1


@pytest.mark.parametrize("n", [2 ** k for k in range(2, 24)])
def test_r2c_forward_matches_oracle(n):
    b = 2 if n >= (1 << 21) else batch_for(n)
    x = real_records(1000 + n, n, b)
    with bf.RealPlan(n, b) as p:
        info = p.info()
        y = p.exec(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    assert info["real"] == 1 and info["n"] == n
    ref = packed_from_full(oracle.records_c64(x.astype(np.complex64), oracle.FORWARD))
    err = oracle.rel_l2(y.cpu().numpy(), ref)
    assert np.all(err <= oracle.tolerance(n)), (n, err.max())
    assert err.max() <= 2e-6, err.max()        # quality band (as for complex records)


# 64..1024: partners by warp shuffle at T = 2..32 threads per record; 2048..8192:
# through shared memory; 2^14: the staged kernel (k_rows_tma); longer: two kernels
@pytest.mark.parametrize("n", [4, 8, 64, 256, 512, 1024, 2048, 4096, 8192, 1 << 14, 1 << 15, 1 << 16, 1 << 20,
                               1 << 23])
def test_c2r_inverse_matches_oracle(n):
    b = 2 if n >= (1 << 21) else 5
    x = real_records(2000 + n, n, b)
    P = packed_from_full(oracle.records_c64(x.astype(np.complex64), oracle.FORWARD)).astype(np.complex64)
    with bf.RealPlan(n, b, bf.FFT_INVERSE) as p:
        z = p.exec(torch.from_numpy(P).cuda())
    torch.cuda.synchronize()
    ref = oracle.records_c64(full_from_packed(P.astype(np.complex128)).astype(np.complex64), oracle.INVERSE)
    # the oracle inverse of a Hermitian spectrum is real (up to rounding of the promotion)
    err = oracle.rel_l2(z.cpu().numpy().astype(np.complex128), ref.real.astype(np.complex128))
    assert np.all(err <= oracle.tolerance(n)), (n, err.max())
    # round trip to the original reals
    assert np.all(oracle.rel_l2(z.cpu().numpy().astype(np.complex128), x.astype(np.complex128))
                  <= oracle.tolerance(n))


@pytest.mark.parametrize("direction", [-1, 1])
@pytest.mark.parametrize("n", [1 << 14, 1 << 15])
def test_real_staged_kernel_reuses_stages(direction, n):
    # 2^14 reals on k_rows_tma, 2^15 on k_rows_tma2: 449 records = three or more
    # per persistent CTA, so every stage / buffer is refilled (R2C split through
    # the exchange buffer; C2R merge from the natural-order staged record)
    b = 449
    x = real_records(3000 + n, n, b)
    full = oracle.records_c64(x.astype(np.complex64), oracle.FORWARD)
    if direction == bf.FFT_FORWARD:
        with bf.RealPlan(n, b) as p:
            y = p.exec(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        err = oracle.rel_l2(y.cpu().numpy(), packed_from_full(full))
    else:
        P = packed_from_full(full).astype(np.complex64)
        with bf.RealPlan(n, b, bf.FFT_INVERSE) as p:
            z = p.exec(torch.from_numpy(P).cuda())
        torch.cuda.synchronize()
        ref = oracle.records_c64(full_from_packed(P.astype(np.complex128)).astype(np.complex64), oracle.INVERSE)
        err = oracle.rel_l2(z.cpu().numpy().astype(np.complex128), ref.real.astype(np.complex128))
    assert np.all(err <= oracle.tolerance(n)), err.max()
    assert err.max() <= 2e-6, err.max()


@pytest.mark.parametrize("n", [1 << 16, 1 << 17, 1 << 18, 1 << 19])
def test_r2c_fused_pipelined_wraps_ring(n):
    # forward records of 2^16..2^19 samples: k_pipe2 with the split fused into its
    # B-tasks (mirrored half tiles).  A batch of 2S + 3 records wraps the L2 ring
    # twice; sampled records (first, last, reused slots, seeded picks) vs the oracle.
    with bf.RealPlan(n, 1) as p:
        info = p.info()
    assert info["kernels_per_exec"] == 1 and info["variant_name"] == "pipe", info
    s = info["ring_records"]
    b = 2 * s + 3
    x = torch.empty((b, n), dtype=torch.float32, device="cuda")
    torch.manual_seed(n)
    x.uniform_(-1, 1)
    with bf.RealPlan(n, b) as p:
        y = p.exec(x)
    torch.cuda.synchronize()
    rows = sorted({0, 1, s - 1, s, s + 1, 2 * s, 2 * s + 1, b - 1})
    xs = x[rows].cpu().numpy()
    ref = packed_from_full(oracle.records_c64(xs.astype(np.complex64), oracle.FORWARD))
    err = oracle.rel_l2(y[rows].cpu().numpy(), ref)
    assert np.all(err <= oracle.tolerance(n)), err.max()
    assert err.max() <= 2e-6, err.max()
    # batch independence: the same records alone
    with bf.RealPlan(n, 1) as p1:
        for i, r in enumerate(rows):
            y1 = p1.exec(x[r:r + 1].contiguous())
            torch.cuda.synchronize()
            assert torch.equal(y1[0], y[r]), r


@pytest.mark.parametrize("n", [1 << 16, 1 << 17, 1 << 19])
def test_c2r_fused_pipelined_wraps_ring(n):
    # inverse records of 2^16..2^19 samples: k_pipe2 with the C2R merge fused into
    # its A-task reads (partners from the packed spectra in HBM / L2).  2S + 3
    # records wrap the ring twice; sampled records vs the oracle's inverse of the
    # Hermitian-extended spectrum, and vs the same records alone.
    with bf.RealPlan(n, 1, bf.FFT_INVERSE) as p:
        info = p.info()
    assert info["kernels_per_exec"] == 1 and info["variant_name"] == "pipe", info
    s = info["ring_records"]
    b = min(2 * s + 3, max(3, (1 << 29) // n))   # at most 2 GiB of spectra
    P = torch.empty((b, n // 2), dtype=torch.complex64, device="cuda")
    torch.manual_seed(n + 1)
    P.view(torch.float32).uniform_(-1, 1)
    with bf.RealPlan(n, b, bf.FFT_INVERSE) as p:
        z = p.exec(P)
    torch.cuda.synchronize()
    rows = sorted({0, 1, min(b - 1, s), min(b - 1, s + 1), min(b - 1, 2 * s + 1), b - 1})
    Ph = P[rows].cpu().numpy()
    ref = oracle.records_c64(full_from_packed(Ph.astype(np.complex128)).astype(np.complex64), oracle.INVERSE)
    err = oracle.rel_l2(z[rows].cpu().numpy().astype(np.complex128), ref.real.astype(np.complex128))
    assert np.all(err <= oracle.tolerance(n)), err.max()
    with bf.RealPlan(n, 1, bf.FFT_INVERSE) as p1:
        for r in rows:
            z1 = p1.exec(P[r:r + 1].contiguous())
            torch.cuda.synchronize()
            assert torch.equal(z1[0], z[r]), r


def test_r2c_closed_forms_and_in_place():
    n = 1024
    j = np.arange(n)
    recs = np.stack([np.eye(1, n, 0)[0], np.ones(n), np.cos(2 * np.pi * 3 * j / n),
                     np.sin(2 * np.pi * 5 * j / n), (-1.0) ** j]).astype(np.float32)
    buf = torch.from_numpy(recs.copy()).cuda()
    with bf.RealPlan(n, 5) as p:
        y = p.exec(buf, buf.view(torch.complex64))   # in place: 4n bytes in, 4n out
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    tol = 1e-5 * np.log2(n) * n
    flat = np.ones(n // 2, complex)
    flat[0] = 1 + 1j                                                            # packed (X[0], X[n/2]) = (1, 1)
    np.testing.assert_allclose(y[0], flat, atol=tol)                            # impulse -> flat
    e = np.zeros(n // 2, complex)
    e[0] = n + 0j
    np.testing.assert_allclose(y[1], e, atol=tol)                               # constant -> (N, 0)
    e[:] = 0
    e[3] = n / 2
    np.testing.assert_allclose(y[2], e, atol=tol)                               # cos tone -> N/2 at bin 3
    e[:] = 0
    e[5] = -1j * n / 2
    np.testing.assert_allclose(y[3], e, atol=tol)                               # sin tone -> -iN/2 at bin 5
    e[:] = 0
    e[0] = 0 + 1j * n                                                           # Nyquist in the packed slot
    np.testing.assert_allclose(y[4], e, atol=tol)


def test_real_plan_errors():
    for n in (2, 3, 1000, 1 << 24):
        with pytest.raises(bf.FFTError) as ei:
            bf.RealPlan(n, 1)
        assert ei.value.code == 1
    with pytest.raises(bf.FFTError) as ei:
        bf.RealPlan(1024, 1, 0)
    assert ei.value.code == 3
    with bf.RealPlan(1024, 2) as p:
        with pytest.raises(ValueError):
            p.exec(torch.zeros((2, 1024), dtype=torch.complex64, device="cuda"))


@pytest.mark.parametrize("n", [1024, 1 << 16])
def test_real_file_stream(tmp_path, n):
    # the paper's record (1024 reals = 4096 bytes) through the file
    # pipeline: R = ceil(bytes / 4n), final record zero-padded, output 4n bytes per record
    r = 37
    x = real_records(77, n, r).reshape(-1)[: r * n - 10]
    src, dst, back = tmp_path / "in.f32", tmp_path / "out.c64", tmp_path / "back.f32"
    x.astype("<f4").tofile(src)
    st = bf.fft_file(str(src), str(dst), n, 1, options=bf.StreamOptions(chunk_bytes=4 * n * 8, real=True))
    assert st["records"] == r and os.path.getsize(dst) == r * 4 * n
    xp = np.zeros(r * n, np.float32)
    xp[: x.size] = x
    ref = packed_from_full(oracle.records_c64(xp.reshape(r, n).astype(np.complex64), oracle.FORWARD))
    y = np.fromfile(dst, "<c8").reshape(r, n // 2)
    assert np.all(oracle.rel_l2(y, ref) <= oracle.tolerance(n))
    with bf.RealPlan(n, r) as p:                   # streamed == in-HBM, bit for bit
        yd = p.exec(torch.from_numpy(xp.reshape(r, n)).cuda()).cpu().numpy()
    assert np.array_equal(yd, y)
    bf.fft_file(str(dst), str(back), n, 1, direction=bf.FFT_INVERSE,
                options=bf.StreamOptions(chunk_bytes=4 * n * 5, real=True))
    z = np.fromfile(back, "<f4").reshape(r, n)
    assert np.all(oracle.rel_l2(z.astype(np.complex128), xp.reshape(r, n).astype(np.complex128))
                  <= oracle.tolerance(n))


def test_real_host_stream_halves_bytes():
    n, r = 1024, 4096
    x = real_records(5, n, r)
    h = bf.HostBuffer(r, n // 2, 0)                # 4n bytes per record, viewed as complex64
    o = bf.HostBuffer(r, n // 2, 0)
    h.a.view(np.float32)[:] = x
    st = bf.exec_host(h.a, n, bf.FFT_FORWARD, 0, out=o.a, options=bf.StreamOptions(real=True, chunk_bytes=4 * n * 512))
    assert st["bytes_in"] == r * 4 * n and st["bytes_out"] == r * 4 * n
    with bf.RealPlan(n, r) as p:
        yd = p.exec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(yd, o.a)
    h.close()
    o.close()
