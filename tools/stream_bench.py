"""Out-of-core streamer measurements (BASELINE.json configs[3] analogue).

A 1 TiB file does not fit on the GPU box's disk, so this measures, per GPU:
  1. the host-link roofline: pinned cudaMemcpyAsync H2D alone, D2H alone, and
     both directions concurrently (the streamer's bound);
  2. a logical multi-GiB stream through fft_exec_host (pinned host source and
     sink, 1024-point records as in PAPER.md:49) — "host-memory source/sink,
     disk excluded";
  3. fft_file on a real on-disk file (page cache hot), the paper's actual
     file -> file path.
Run one process per GPU (torchrun) to measure concurrent GPUs sharing the host.
Prints one JSON line per rank.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402
from synth import gpu as sg  # noqa: E402


def gbps(nbytes, s):
    return nbytes / s / 1e9


def link_probe(dev, nbytes):
    h1 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {}
    for name, ops in (("h2d", [(s1, d1, h1)]), ("d2h", [(s2, h2, d2)]),
                      ("both", [(s1, d1, h1), (s2, h2, d2)])):
        for _ in range(2):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for st, dst, src in ops:
                with torch.cuda.stream(st):
                    dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize(dev)
            el = time.perf_counter() - t0
        res[name + "_GBps"] = gbps(nbytes * len(ops), el) / (len(ops) if name == "both" else 1)
    return res   # "both" = per direction while both run


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--buf-gib", type=float, default=4.0)
    ap.add_argument("--passes", type=int, default=8)
    ap.add_argument("--file-gib", type=float, default=8.0)
    ap.add_argument("--dir", default="/tmp")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    out = {"rank": rank, "world": world, "n": a.n}
    out["link"] = link_probe(dev, 1 << 30)

    # logical stream through the host streamer
    nbytes = int(a.buf_gib * 2 ** 30) // (8 * a.n) * (8 * a.n)
    rec = nbytes // (8 * a.n)
    d = torch.empty(rec * a.n, dtype=torch.complex64, device=dev)
    sg.fill_random(d, 7, first_sample=rank * rec * a.n)
    h = torch.empty_like(d, device="cpu").pin_memory()
    h.copy_(d)
    del d
    torch.cuda.empty_cache()
    bf.exec_host(h, a.n, bf.FFT_FORWARD, local)                 # warm (cached resources)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    stats = None
    for _ in range(a.passes):
        stats = bf.exec_host(h, a.n, bf.FFT_FORWARD, local)     # in place
    el = time.perf_counter() - t0
    out["stream"] = {"logical_GiB": a.passes * nbytes / 2 ** 30, "records": a.passes * rec,
                     "records_per_s": a.passes * rec / el, "GBps_each_way": gbps(a.passes * nbytes, el),
                     "last_pass": stats}

    # a real file on disk (page cache hot after the write); rank 0 runs the
    # library's own multi-GPU file path over every visible GPU
    if a.file_gib > 0 and rank == 0:
        ng = torch.cuda.device_count()
        fb = int(a.file_gib * 2 ** 30) // (8 * a.n) * (8 * a.n)
        src = os.path.join(a.dir, f"bfft_in_{rank}.c64")
        dst = os.path.join(a.dir, f"bfft_out_{rank}.c64")
        with open(src, "wb") as f:
            left = fb
            view = h.numpy().view("uint8")
            while left > 0:
                k = min(left, view.size)
                f.write(view[:k])
                left -= k
        res = {}
        for g in sorted({1, ng}):
            bf.fft_file(src, dst, a.n, g)                        # warm
            os.remove(dst)                                       # time a fresh output file
            t0 = time.perf_counter()
            st = bf.fft_file(src, dst, a.n, g)
            el = time.perf_counter() - t0
            res[f"ngpu{g}"] = {"wall_s": el, "file_GBps": gbps(fb, el), "stats": st}
        out["file"] = {"GiB": fb / 2 ** 30, "runs": res,
                       "note": "page cache hot; pread/pwrite through the host page cache"}
        os.remove(src)
        os.remove(dst)
    if world > 1:
        dist.barrier()
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
