"""Config 4 (BASELINE.json configs[3]): a 1 TiB logical signal
streamed host -> GPU -> host with copy/compute overlap, at G = 1, 2, 4 GPUs of
one box, against the measured host-link roofline at the same G.

Source and sink are host-memory rings (fft_stream_host: the 1 TiB stream is
replayed from a K-chunk seeded capture ring; outputs go to a rolling ring —
"host-memory source/sink, disk excluded", the survey's (ii) option), pinned
on each GPU's NUMA node (fft_host_alloc).  GPU g streams its contiguous share
of the logical records (fft_partition).  All G streams start together (one
thread per GPU, barrier); the aggregate is total bytes / the slowest GPU.

Roofline at G: every GPU runs fft_link_probe at the same time (H2D and D2H
concurrently, pinned NUMA-local buffers); the stream's fraction is its
per-direction GB/s over that aggregate.

Parity: >= 1 tapped record per GiB of the stream (taps) is checked bit for bit
against the same ring record transformed in HBM (whose parity with the CPU
oracle is tests/test_gpu_parity.py's); the same 1 TiB stream with its taps
checked against the oracle itself is tests/test_gpu_config4.py (this tool
does not touch oracle/: only tests and bench.py's CPU leg may).

  python tools/stream_tib.py [--gpus 1,2,4] [--tib 1.0] [--n 1024] [--json OUT]
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402
import synth  # noqa: E402


def probe(gpus, nbytes, reps=3):
    bufs = {g: (bf.HostBuffer(nbytes // 8, 1, g), bf.HostBuffer(nbytes // 8, 1, g)) for g in gpus}
    res, bar = {}, threading.Barrier(len(gpus))

    def run(g):
        bar.wait()
        res[g] = bf.link_probe(g, bufs[g][0], bufs[g][1], nbytes, reps=reps)
    th = [threading.Thread(target=run, args=(g,)) for g in gpus]
    [t.start() for t in th]
    [t.join() for t in th]
    for a, b in bufs.values():
        a.close()
        b.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", default="1,2,4")
    ap.add_argument("--tib", type=float, default=1.0)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--chunk-mib", type=int, default=256)
    ap.add_argument("--ring-chunks", type=int, default=4)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    n = a.n
    rb = 8 * n
    total_bytes = int(a.tib * 2 ** 40)
    total = total_bytes // rb                       # logical records (2^27 at N = 1024)
    crec = (a.chunk_mib << 20) // rb
    k = crec * a.ring_chunks                        # ring records (input capture ring)
    ndev = torch.cuda.device_count()
    rows = []
    seed = synth.DEFAULT_SEED
    ring_h = synth.random_records(seed, n, 0, k)    # ring record j = seeded record j
    # in-HBM reference of the ring (bit-identity of every tap)
    ref = {}
    for gcount in [int(x) for x in a.gpus.split(",")]:
        if gcount > ndev:
            rows.append({"gpus": gcount, "skipped": f"only {ndev} GPUs visible"})
            continue
        gpus = list(range(gcount))
        link = probe(gpus, 1 << 30)                   # burst: best of 3 concurrent rounds
        link_sus = probe(gpus, 1 << 30, reps=200)     # sustained: ~5-10 s of back-to-back rounds
        ins, outs, opts, stats = {}, {}, {}, {}
        # taps: one record per GiB of the whole logical stream, in each GPU's share
        tap_all = np.arange(0, total, (1 << 30) // rb, dtype=np.int64)
        for g in gpus:
            if g not in ref:
                x = torch.from_numpy(ring_h).cuda(g)
                with torch.cuda.device(g):
                    with bf.Plan(n, k, device=g) as p:
                        ref[g] = p.exec(x, torch.empty_like(x)).cpu().numpy()
                    torch.cuda.synchronize()
                del x
            ins[g] = bf.HostBuffer(k, n, g)
            ins[g].a[:] = ring_h
            outs[g] = bf.HostBuffer(k, n, g)
        # contiguous shares (fft_partition's rule, rounded to whole rings so GPU g's
        # local record i is global record first + i and reads ring record i mod k)
        per = (total // gcount) // k * k
        shares = {g: (g * per, per if g < gcount - 1 else total - g * per) for g in gpus}
        res, bar = {}, threading.Barrier(gcount)

        def run(g):
            first, count = shares[g]
            taps = tap_all[(tap_all >= first) & (tap_all < first + count)] - first
            o = bf.StreamOptions(n=n, chunk_bytes=crec * rb, taps=taps, timeline=64)
            opts[g] = (o, taps + first)
            bar.wait()
            t0 = time.perf_counter()
            st = bf.stream_host(ins[g].a, outs[g].a, n, count, device=g, options=o)
            res[g] = (st, time.perf_counter() - t0)

        th = [threading.Thread(target=run, args=(g,)) for g in gpus]
        t0 = time.perf_counter()
        [t.start() for t in th]
        [t.join() for t in th]
        wall = time.perf_counter() - t0
        slowest = max(res[g][1] for g in gpus)
        moved = sum(res[g][0]["bytes_in"] for g in gpus)
        # parity: every tap bit-identical to the in-HBM transform of its ring record
        bad, ntaps = 0, 0
        for g in gpus:
            o, glob = opts[g]
            rid = glob % k
            bad += int(np.sum([not np.array_equal(o.tap_out[j], ref[g][rid[j]]) for j in range(len(rid))]))
            ntaps += len(rid)
        agg_h2d = sum(link[g]["both_h2d"] for g in gpus)
        agg_d2h = sum(link[g]["both_d2h"] for g in gpus)
        agg_sus = sum(link_sus[g]["both_sustained"] for g in gpus)
        each_way = moved / slowest / 1e9
        row = {"gpus": gcount, "n": n, "logical_bytes": total * rb, "records": total, "seconds": slowest,
               "wall_s": wall, "records_per_s": total / slowest, "GBps_each_way": each_way,
               "link_roofline": {"per_gpu": link, "aggregate_concurrent_h2d": agg_h2d,
                                 "aggregate_concurrent_d2h": agg_d2h},
               "link_sustained": {"per_gpu": {g: link_sus[g]["both_sustained"] for g in gpus},
                                  "aggregate_each_way": agg_sus},
               "frac_of_link_h2d": each_way / agg_h2d, "frac_of_link_d2h": each_way / agg_d2h,
               "frac_of_sustained_link": each_way / agg_sus,
               "numa_nodes": {g: res[g][0]["numa_node"] for g in gpus},
               "busy": {g: {s: res[g][0][s] / res[g][1] for s in ("h2d_s", "fft_s", "d2h_s")} for g in gpus},
               "taps": ntaps, "taps_not_bit_identical": bad,
               "timeline_gpu0": opts[0][0].timeline_out[:8].round(5).tolist()}
        rows.append(row)
        print(json.dumps({kk: v for kk, v in row.items() if kk != "timeline_gpu0"}), flush=True)
        for g in gpus:
            ins[g].close()
            outs[g].close()
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
