"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
include/blockfft.h declares, validates arguments with SPEC-style messages, and
the partitioner reproduces the paper's record/block arithmetic.  No compute
call is made (there is no GPU here)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT, read_golden

import paper_1407_6915_b200 as bf
from paper_1407_6915_b200 import _abi


def header_functions():
    src = open(os.path.join(ROOT, "include", "blockfft.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fft_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported():
    names = header_functions()
    assert len(names) >= 13
    lib = ctypes.CDLL(_abi.LIB_PATH)
    for name in names:
        assert hasattr(lib, name), f"{name} declared in blockfft.h but not exported"
    assert sorted(_abi.EXPORTED) == names


def test_library_is_sm100a_only():
    # the fatbin must carry sm_100a SASS (cuobjdump is in the image)
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(7|8|9)\d", out)


def test_version():
    assert bf.version() == 1


@pytest.mark.parametrize("n", [0, 1, 3, 1000, 6, 1 << 23, -4])
def test_plan_rejects_unsupported_size(n):
    # "unsupported transform size" naming the offending value
    with pytest.raises(bf.FFTError) as ei:
        bf.Plan(n, 1)
    assert ei.value.code == _abi.FFT_E_SIZE
    assert f"unsupported transform size: {n}" in str(ei.value)


def test_plan_rejects_batch_and_direction():
    with pytest.raises(bf.FFTError) as ei:
        bf.Plan(1024, 0)
    assert ei.value.code == _abi.FFT_E_BATCH and "batch must be >= 1: 0" in str(ei.value)
    with pytest.raises(bf.FFTError) as ei:
        bf.Plan(1024, 4, direction=2)
    assert ei.value.code == _abi.FFT_E_DIR and "direction must be -1 or +1: 2" in str(ei.value)


def test_plan_create_rejects_direction_zero():
    # fft_plan_create(n, b, 0) is FFT_E_DIR; identity (dir 0) is reachable
    # only through an explicit FFT_VARIANT_IDENTITY, which in turn takes only dir 0
    lib = _abi.lib
    assert not lib.fft_plan_create(1024, 4, 0)
    assert lib.fft_last_status() == _abi.FFT_E_DIR
    assert "direction must be -1 or +1: 0" in bf.last_error()
    assert not lib.fft_plan_create_ex(1024, 4, 0, _abi.VARIANT_AUTO)
    assert lib.fft_last_status() == _abi.FFT_E_DIR
    assert not lib.fft_plan_create_ex(1024, 4, -1, _abi.VARIANT_IDENTITY)
    assert lib.fft_last_status() == _abi.FFT_E_DIR


def test_plan_options_validated_without_gpu():
    lib = _abi.lib
    for field, val in (("variant", 9), ("impl", -1), ("config", -2), ("cluster_size", -1),
                       ("ring_records", -5), ("ring_lag", -1)):
        o = _abi.PlanOpts()
        setattr(o, field, val)
        assert not lib.fft_plan_create_opts(1024, 1, -1, ctypes.byref(o))
        assert lib.fft_last_status() == _abi.FFT_E_ARG, field
        assert f"{field}={val}" in bf.last_error()


def test_exec_null_plan_is_arg_error():
    lib = _abi.lib
    assert lib.fft_exec(None, None, None, None) == _abi.FFT_E_ARG
    assert lib.fft_plan_get_info(None, None) == _abi.FFT_E_ARG
    lib.fft_plan_destroy(None)  # NULL-safe


@pytest.mark.parametrize("row", read_golden("paper_record_arithmetic.txt"), ids=lambda r: r[0])
def test_record_arithmetic_golden(row):
    name, file_bytes, rec_bytes, block_bytes, exp_rec, exp_blocks, exp_pad, _ = row
    file_bytes, rec_bytes, block_bytes = int(file_bytes), int(rec_bytes), int(block_bytes)
    # our records are complex64: record_len N points = 8N bytes
    n = rec_bytes // 8
    r = bf.file_records(file_bytes, n)
    assert r == int(exp_rec)
    # the paper's blocks: records grouped into block_bytes-sized map tasks
    per_block = block_bytes // rec_bytes
    blocks = -(-r // per_block)
    assert blocks == int(exp_blocks)
    # zero padding of the final record, in 4-byte real samples
    assert (r * rec_bytes - file_bytes) // 4 == int(exp_pad)


def test_paper_2048_map_tasks_as_partition():
    # 2^40 B in 512 MB blocks -> 2,048 map tasks of equal size.
    r = bf.file_records(1 << 40, 512)           # 4096-byte records
    assert r == 268435456
    for g in (0, 1, 1023, 2047):
        f, c = bf.partition(r, 2048, g)
        assert c == 131072 and f == g * 131072


def test_file_records_errors():
    with pytest.raises(bf.FFTError) as ei:
        bf.file_records(0, 1024)
    assert ei.value.code == _abi.FFT_E_EMPTY
    with pytest.raises(bf.FFTError) as ei:
        bf.file_records(12, 1024)
    assert ei.value.code == _abi.FFT_E_ARG
    with pytest.raises(bf.FFTError) as ei:
        bf.file_records(8192, 1000)
    assert ei.value.code == _abi.FFT_E_SIZE
    assert bf.file_records(8, 1024) == 1
    assert bf.file_records(8192 + 8, 1024) == 2


@pytest.mark.parametrize("total,g", [(0, 3), (1, 8), (7, 8), (100, 8), (134217728, 8),
                                     (2 ** 40 // 8 + 5, 8), (2 ** 62 + 3, 7)])
def test_partition_contiguous_cover(total, g):
    prev_end = 0
    sizes = []
    for p in range(g):
        f, c = bf.partition(total, g, p)
        assert f == prev_end and c >= 0
        assert f == (p * total) // g            # floor(g R / G), exact in Python ints
        prev_end = f + c
        sizes.append(c)
    assert prev_end == total
    assert max(sizes) - min(sizes) <= 1


def test_partition_errors():
    for args in [(10, 0, 0), (10, 2, 2), (10, 2, -1), (-1, 2, 0)]:
        with pytest.raises(bf.FFTError) as ei:
            bf.partition(*args)
        assert ei.value.code == _abi.FFT_E_ARG


def test_fft_file_validation_without_gpu(tmp_path):
    p = tmp_path / "x.c64"
    p.write_bytes(b"\0" * 64)
    with pytest.raises(bf.FFTError) as ei:
        bf.fft_file(str(p), str(tmp_path / "y"), 1000, 1)
    assert ei.value.code == _abi.FFT_E_SIZE
    assert not os.path.exists(str(tmp_path / "y.tmp"))
