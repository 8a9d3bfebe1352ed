"""One-process-per-GPU (or per node) plumbing for the record-parallel path
(SURVEY.md §8(e), §8(f) NEXT-3).

Records are independent, so the data path has no collective: rank g owns the
contiguous record range ``fft_partition(R, G, g)`` (the C ABI's partitioner,
PAPER.md:53 one block per map task) and ``fft_file_range`` writes its outputs
at byte offset ``first * 8 N`` of one shared, pre-sized file (PAPER.md:63 zero
reducers, outputs named by position).  The only cross-rank operations are
plumbing over torch.distributed (NCCL on GPUs, gloo on CPU or across nodes):
barriers, an error flag, and the max of per-rank times.  ``bench.py`` uses
``rank_info`` / ``max_over_ranks``; ``fan_out`` is the multi-node form of
``fft_file`` (the paper's Hadoop fan-out over EC2 nodes, PAPER.md:111-115,
without HDFS, map tasks or -getmerge).
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class RankInfo:
    rank: int
    world: int
    local_rank: int


def rank_info() -> RankInfo:
    """RANK / WORLD_SIZE / LOCAL_RANK from the torchrun environment (defaults: single process)."""
    return RankInfo(int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
                    int(os.environ.get("LOCAL_RANK", 0)))


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def my_records(total_records: int, info: RankInfo | None = None) -> tuple[int, int]:
    """(first, count) of this rank's contiguous record range."""
    from . import partition
    info = info or rank_info()
    return partition(total_records, info.world, info.rank)


def _all_reduce(value: float, op: str, device=None) -> float:
    d = _dist()
    if d is None or d.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    d.all_reduce(t, op=d.ReduceOp.MAX if op == "max" else d.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over the process group (timings: the slowest rank)."""
    return _all_reduce(value, "max", device)


def sum_over_ranks(value: float, device=None) -> float:
    return _all_reduce(value, "sum", device)


def barrier(device=None) -> None:
    d = _dist()
    if d is not None and d.get_world_size() > 1:
        if device is not None and d.get_backend() == "nccl":
            d.barrier(device_ids=[device.index if hasattr(device, "index") else int(device)])
        else:
            d.barrier()


def fan_out(in_path: str, out_path: str, record_len: int, direction: int = -1, device: int | None = None,
            options=None, transform=None, reduce_device=None) -> dict:
    """Every rank of the process group transforms its contiguous record range of
    ``in_path`` into one shared output.

    Rank 0 creates ``out_path + ".tmp"`` pre-sized to R*8N bytes; after a
    barrier each rank runs ``transform(in_path, tmp, record_len, first, count,
    device, direction, options)`` — by default ``fft_file_range`` on its local
    GPU, which writes the range at its own byte offset; the ranks agree on
    success through one max-reduction of an error flag, and rank 0 renames the
    file or removes it on any rank's failure.
    Returns this rank's stats (``first``, ``count`` added); raises on failure
    on every rank.  ``transform`` is injectable so the coordination is testable
    on CPU (tests/test_dist.py); the GPU path is tests/test_gpu_dist.py.
    """
    from . import FFTError, file_range, file_records
    info = rank_info()
    if device is None:
        device = info.local_rank
    total = file_records(os.path.getsize(in_path), record_len)
    tmp = out_path + ".tmp"
    err = 0.0
    if info.rank == 0:
        try:
            with open(tmp, "wb") as f:
                f.truncate(total * 8 * record_len)
        except OSError:
            err = 1.0
    if max_over_ranks(err, reduce_device):
        raise FFTError(8, f"cannot create {tmp}")
    first, count = my_records(total, info)
    fn = transform or (lambda i, o, n, f, c, dev, d, opt: file_range(i, o, n, f, c, dev, d, opt))
    stats, msg = {}, ""
    try:
        stats = fn(in_path, tmp, record_len, first, count, device, direction, options) or {}
    except Exception as e:       # noqa: BLE001 — every rank must reach the agreement below
        err, msg = 1.0, str(e)
    failed = max_over_ranks(err, reduce_device) > 0
    if info.rank == 0:
        if failed:
            try:
                os.unlink(tmp)
            except OSError:
                pass
        else:
            os.replace(tmp, out_path)
    barrier(reduce_device)
    if failed:
        raise FFTError(8, f"fan_out failed on some rank (this rank: {msg or 'ok'})")
    stats = dict(stats)
    stats.update(first=first, count=count, rank=info.rank, world=info.world)
    return stats
