"""The multi-process file path on the GPU:
two ranks (gloo for the plumbing) each run ``fft_file_range`` through the C
streamer on their record range of one file — both on cuda:0 here, since the
ranges are independent kernels that never wait on each other — and
``dist.fan_out`` assembles one output that is bit-identical to ``fft_file``
on the whole file, and within the north_star bar of the oracle."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
bf = pytest.importorskip("paper_1407_6915_b200")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, pin, pout, n, q):
    import torch.distributed as dist
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1407_6915_b200 as bfl
        from paper_1407_6915_b200 import dist as bd
        st = bd.fan_out(pin, pout, n, device=0, options=bfl.StreamOptions(chunk_bytes=8 * n * 5))
        q.put((rank, st, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, str(e)))
    finally:
        dist.destroy_process_group()


def test_two_process_fan_out_matches_fft_file(tmp_path):
    import torch.multiprocessing as mp
    n, r = 2048, 21
    s = synth.random_samples(61, 0, r * n - 3)
    pin, pout, whole = tmp_path / "in", tmp_path / "out", tmp_path / "whole"
    s.astype("<c8").tofile(pin)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, str(pin), str(pout), n, q)) for k in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    assert all(e is None for _, _, e in res), res
    assert sum(st["records"] for _, st, _ in res) == r
    bf.fft_file(str(pin), str(whole), n, 1)
    assert pout.read_bytes() == whole.read_bytes()
    y = np.fromfile(pout, dtype="<c8").reshape(-1, n)
    assert np.all(oracle.rel_l2(y, oracle.file_transform(pin.read_bytes(), n)) <= oracle.tolerance(n))
