"""Multi-process (world_size 2, gloo, CPU) tests of the record-parallel host
logic of ``paper_1407_6915_b200.dist.fan_out``:
every rank derives its own contiguous record range from the C-ABI
partitioner, ranges tile the file exactly, rank 0 pre-sizes one shared output,
each rank writes its range at its byte offset (no merge, no collective on the
data), the ranks agree on success, rank 0 renames — or removes the temporary
on any rank's failure — and the timing reduction takes the max over ranks.

The CPU has no kernels, so the per-rank transform is injected: a positional
byte copy (the identity).  The default transform, ``fft_file_range`` through
the C streamer, runs the same coordination on the GPU in
tests/test_gpu_dist.py."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _copy_range(i, o, n, first, count, device, direction, options, fail_rank=None):
    """Identity 'transform' of records [first, first+count) at their offsets."""
    if fail_rank is not None and int(os.environ["RANK"]) == fail_rank:
        raise RuntimeError("injected failure")
    rb = 8 * n
    size = os.path.getsize(i)
    with open(i, "rb") as fi:
        fi.seek(first * rb)
        data = fi.read(count * rb)
    data += b"\0" * (count * rb - len(data))           # zero-padded tail (reading c6)
    fd = os.open(o, os.O_WRONLY)
    try:
        os.pwrite(fd, data, first * rb)
    finally:
        os.close(fd)
    return {"records": count, "size": size}


def _worker(rank, world, port, path_in, path_out, n, fail_rank, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1407_6915_b200 import dist as bd
        err = None
        st = None
        try:
            st = bd.fan_out(path_in, path_out, n, transform=lambda *a: _copy_range(*a, fail_rank=fail_rank))
        except Exception as e:   # noqa: BLE001
            err = str(e)
        t = bd.max_over_ranks(float(rank + 1) * 0.5)
        got = [None] * world
        dist.all_gather_object(got, (st or {}).get("first"), )
        q.put((rank, st, err, t, got))
    finally:
        dist.destroy_process_group()


def _run(world, n, samples, fail_rank=None):
    d = tempfile.mkdtemp()
    pin, pout = os.path.join(d, "in.c64"), os.path.join(d, "out.c64")
    samples.astype("<c8").tofile(pin)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, pin, pout, n, fail_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return pin, pout, res


@pytest.mark.parametrize("world,total", [(2, 37), (2, 1), (2, 1024)])
def test_two_ranks_fan_out(world, total):
    n = 64
    data = synth.random_samples(3, 0, total * n - 5)       # ragged tail: last record zero-padded
    pin, pout, res = _run(world, n, data)
    assert all(r[2] is None for r in res), res
    ranges = [(r[1]["first"], r[1]["count"]) for r in res]
    assert ranges[0][0] == 0 and sum(c for _, c in ranges) == total
    for (f0, c0), (f1, _) in zip(ranges, ranges[1:]):
        assert f0 + c0 == f1                            # contiguous, disjoint
    assert all(r[3] == 0.5 * world for r in res)        # max over ranks
    out = open(pout, "rb").read()
    assert len(out) == total * 8 * n                    # pre-sized R*8N
    assert out == open(pin, "rb").read() + b"\0" * 40   # file order restored, no merge
    assert not os.path.exists(pout + ".tmp")


def test_fan_out_failure_on_one_rank_removes_tmp():
    n, total = 64, 10
    pin, pout, res = _run(2, n, synth.random_samples(4, 0, total * n), fail_rank=1)
    assert all(r[2] is not None for r in res)           # every rank raises
    assert "injected failure" in res[1][2]
    assert not os.path.exists(pout) and not os.path.exists(pout + ".tmp")
