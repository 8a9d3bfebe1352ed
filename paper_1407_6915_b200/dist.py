"""One-process-per-GPU plumbing for the record-parallel path.

Records are independent, so the data path has no collective: rank g owns the
contiguous record range ``fft_partition(R, G, g)`` (the C ABI's partitioner,
PAPER.md:53 one block per map task) and writes its outputs at byte offset
``first * 8 N`` (PAPER.md:63 zero reducers, outputs named by position).  The
only cross-rank operations are plumbing: a start/stop barrier and the max of
the per-rank device times (torch.distributed; NCCL on GPUs, gloo on CPU).
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RankInfo:
    rank: int
    world: int
    local_rank: int


def rank_info() -> RankInfo:
    """RANK / WORLD_SIZE / LOCAL_RANK from the torchrun environment (defaults: single process)."""
    return RankInfo(int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
                    int(os.environ.get("LOCAL_RANK", 0)))


def my_records(total_records: int, info: RankInfo | None = None) -> tuple[int, int]:
    """(first, count) of this rank's contiguous record range."""
    from . import partition
    info = info or rank_info()
    return partition(total_records, info.world, info.rank)


def write_at_offset(path: str, first_record: int, record_len: int, data) -> None:
    """Write this rank's output records into the shared, pre-sized output file at
    byte offset first_record * 8 * record_len (no merge step, no collective)."""
    buf = np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    fd = os.open(path, os.O_WRONLY)
    try:
        off = first_record * 8 * record_len
        done = 0
        while done < buf.size:
            done += os.pwrite(fd, buf[done:], off + done)
    finally:
        os.close(fd)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over the process group (timings: the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
