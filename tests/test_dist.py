"""Multi-process (world_size 2, gloo, CPU) tests of the record-parallel host
logic: every rank derives its own contiguous record range from the C-ABI
partitioner, ranges tile the file exactly, each rank writes its outputs at its
byte offset into one pre-sized file (no merge, no collective), and the timing
reduction takes the max over ranks."""
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


def _worker(rank, world, port, path_in, path_out, n, total, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1407_6915_b200 import dist as bd
        info = bd.rank_info()
        first, count = bd.my_records(total, info)
        # rank-local "transform": the identity (the CPU has no kernels); the
        # point under test is partition + offset writes reproducing file order
        x = np.fromfile(path_in, dtype="<c8", count=count * n, offset=first * 8 * n)
        bd.write_at_offset(path_out, first, n, x)
        t = bd.max_over_ranks(float(rank + 1) * 0.5)
        got = [None] * world
        dist.all_gather_object(got, (first, count))
        q.put((rank, first, count, t, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total", [(2, 37), (2, 1), (2, 1024)])
def test_two_ranks_partition_and_offset_writes(world, total):
    n = 64
    with tempfile.TemporaryDirectory() as d:
        pin, pout = os.path.join(d, "in.c64"), os.path.join(d, "out.c64")
        data = synth.random_samples(3, 0, total * n)
        data.astype("<c8").tofile(pin)
        with open(pout, "wb") as f:
            f.truncate(total * n * 8)           # pre-sized output (fft_file does the same)
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, pin, pout, n, total, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = [q.get(timeout=120) for _ in range(world)]
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        res.sort()
        ranges = res[0][4]
        assert all(r[4] == ranges for r in res)          # every rank sees the same plan
        assert ranges[0][0] == 0 and sum(c for _, c in ranges) == total
        for (f0, c0), (f1, _) in zip(ranges, ranges[1:]):
            assert f0 + c0 == f1                            # contiguous, disjoint
        assert all(r[3] == 0.5 * world for r in res)        # max over ranks
        assert open(pout, "rb").read() == open(pin, "rb").read()   # file order restored, no merge
