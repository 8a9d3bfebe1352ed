"""The command line (python -m paper_1407_6915_b200): validation exit codes and
the partition plan on CPU; the file transform itself on the GPU, checked against
the oracle (SURVEY.md §8(b) CLI exit codes; SPEC.md "Invariants")."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    e["PYTHONPATH"] = ROOT + os.pathsep + e.get("PYTHONPATH", "")
    p = subprocess.run([sys.executable, "-m", "paper_1407_6915_b200", *args], capture_output=True, text=True,
                       env=e, cwd=ROOT, timeout=300)
    return p.returncode, p.stdout, p.stderr


def test_cli_partition_plan():
    rc, out, _ = run_cli("partition", "--records", "37", "--gpus", "4")
    assert rc == 0
    d = json.loads(out)
    got = [(r["first"], r["count"]) for r in d["ranges"]]
    assert got == [(g * 37 // 4, (g + 1) * 37 // 4 - g * 37 // 4) for g in range(4)]


def test_cli_validation_exit_codes(tmp_path):
    src = tmp_path / "in.c64"
    np.zeros(64, np.complex64).tofile(src)
    rc, _, err = run_cli("fft", str(src), str(tmp_path / "o1"), "--record-len", "1000")
    assert rc == 1 and "unsupported transform size: 1000" in err
    rc, _, _ = run_cli("fft", str(src), str(tmp_path / "o2"))                  # missing --record-len
    assert rc == 1
    existing = tmp_path / "exists"
    existing.write_bytes(b"x")
    rc, _, err = run_cli("fft", str(src), str(existing), "--record-len", "16")
    assert rc == 1 and "--force" in err and existing.read_bytes() == b"x"
    rc, _, _ = run_cli("fft", str(src), str(tmp_path / "o3"), "--record-len", "16",
                       env={"BLOCKFFT_BLOCK_SIZE": "lots"})
    assert rc == 1


@pytest.mark.gpu
def test_cli_file_transform_and_io_errors(tmp_path):
    n, r = 1024, 7
    s = synth.random_samples(19, 0, n * r + 300)          # ragged tail: final record zero-padded
    src, dst = tmp_path / "in.c64", tmp_path / "out.c64"
    s.astype("<c8").tofile(src)
    rc, out, err = run_cli("fft", str(src), str(dst), "--record-len", str(n), "--chunk-bytes", str(8 * n * 3))
    assert rc == 0, err
    assert json.loads(out)["stats"]["records"] == r + 1
    y = np.fromfile(dst, dtype="<c8").reshape(-1, n)
    ref = oracle.file_transform(src.read_bytes(), n)
    assert np.all(oracle.rel_l2(y, ref) <= oracle.tolerance(n))
    back = tmp_path / "back.c64"
    rc, _, err = run_cli("fft", str(dst), str(back), "--record-len", str(n), "--inverse",
                         env={"BLOCKFFT_BLOCK_SIZE": str(8 * n * 2)})
    assert rc == 0, err
    z = np.fromfile(back, dtype="<c8").reshape(-1, n)
    padded = np.zeros((r + 1) * n, np.complex64)
    padded[: s.size] = s
    assert np.all(oracle.rel_l2(z, padded.reshape(-1, n)) <= 2 * oracle.tolerance(n))
    rc, _, err = run_cli("fft", str(tmp_path / "missing"), str(tmp_path / "o"), "--record-len", str(n))
    assert rc == 3 and "cannot open" in err
    rc, _, _ = run_cli("fft", str(src), str(tmp_path / "o4"), "--record-len", str(n), "--ngpu", "99")
    assert rc == 2


@pytest.mark.gpu
def test_cli_real_and_stft(tmp_path):
    n = 1024
    x = synth.random_samples(23, 0, 9 * n // 2).view(np.float32)
    src, dst = tmp_path / "in.f32", tmp_path / "out.c64"
    x.astype("<f4").tofile(src)
    rc, out, err = run_cli("fft", str(src), str(dst), "--record-len", str(n), "--real")
    assert rc == 0, err
    y = np.fromfile(dst, "<c8").reshape(-1, n // 2)
    full = oracle.records_c64(x.reshape(-1, n).astype(np.complex64), oracle.FORWARD)
    packed = full[:, : n // 2].copy()
    packed[:, 0] = full[:, 0].real + 1j * full[:, n // 2].real
    assert np.all(oracle.rel_l2(y, packed) <= oracle.tolerance(n))
    sig = synth.random_samples(29, 0, 5000)
    s2, d2 = tmp_path / "sig.c64", tmp_path / "stft.c64"
    sig.astype("<c8").tofile(s2)
    rc, out, err = run_cli("fft", str(s2), str(d2), "--record-len", "256", "--hop", "128", "--window", "hann")
    assert rc == 0, err
    assert json.loads(out)["stats"]["records"] == 1 + -(-(5000 - 256) // 128)
    rc, _, err = run_cli("fft", str(s2), str(tmp_path / "bad"), "--record-len", "256", "--hop", "128", "--identity")
    assert rc == 1


@pytest.mark.gpu
def test_cli_fan_out_single_process(tmp_path):
    n = 2048
    s = synth.random_samples(37, 0, 11 * n)
    src, dst, ref = tmp_path / "in.c64", tmp_path / "out.c64", tmp_path / "ref.c64"
    s.astype("<c8").tofile(src)
    rc, out, err = run_cli("fan-out", str(src), str(dst), "--record-len", str(n))
    assert rc == 0, err
    assert json.loads(out)["count"] == 11
    rc, _, err = run_cli("fft", str(src), str(ref), "--record-len", str(n))
    assert rc == 0 and dst.read_bytes() == ref.read_bytes()
