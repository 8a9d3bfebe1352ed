"""Config 5 (BASELINE.json configs[4]): record-length sweep
2^8..2^22, forward AND inverse, 4 GiB of records per N (in HBM, out of
place, inputs >> L2), the default (AUTO) plan: CUDA-event time of one
fft_exec (best of 10 after 3 warm-ups), algorithmic GB/s (16 N bytes per
record) and its fraction of the measured HBM copy bandwidth; with --ncu-csv
(the launch list of tools/ncu_sweep_target.py under ncu) the DRAM bytes per
launch and their ratio to the algorithmic bytes.

  python tools/sweep.py [--min 8] [--max 22] [--gib 4] [--ncu-csv F] [--json OUT]
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse_ncu(path, lo, hi):
    """Per-N DRAM bytes of the measured (second) launch of each N, in order."""
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[hdr_i]
    ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), \
        hdr.index("Metric Unit")
    iid = hdr.index("ID")
    launches = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv:
            continue
        d = launches.setdefault(int(r[iid]), {"kernel": r[ik]})
        d[r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    ours = ("k_rows", "k_pipe", "k_cluster", "k_fs_", "k_copy")
    ordered = [launches[i] for i in sorted(launches) if any(o in launches[i]["kernel"] for o in ours)]
    out = {}
    for j, k in enumerate(range(lo, hi + 1)):
        if 2 * j + 1 < len(ordered):
            out[k] = ordered[2 * j + 1]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min", type=int, default=8)
    ap.add_argument("--max", type=int, default=22)
    ap.add_argument("--gib", type=float, default=4.0)
    ap.add_argument("--ncu-csv", default=None)
    ap.add_argument("--json", default=None)
    ap.add_argument("--merge", default=None, help="add the ncu DRAM bytes to the rows of an earlier --json run")
    a = ap.parse_args()
    ncu = parse_ncu(a.ncu_csv, a.min, a.max) if a.ncu_csv else {}
    rows = []
    if a.merge:
        rows = json.load(open(a.merge))["rows"]
        for row in rows:
            m = ncu.get(row["log2n"])
            if m and row["dir"] == -1:
                tr = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                row.update(ncu_kernel=m["kernel"][:60], ncu_dram_bytes=tr,
                           ncu_traffic_ratio=tr / (16.0 * row["n"] * row["batch"]),
                           ncu_ms=m.get("gpu__time_duration.sum", 0) * 1e3)
            print(f"N=2^{row['log2n']:<2} dir={row['dir']:+d} {row['variant']:>6} {row['ms']:7.3f} ms "
                  f"{row['alg_GBps']:7.1f} GB/s {row['frac']:6.1%}" +
                  (f"  ncu DRAM {row['ncu_traffic_ratio']:.3f}x alg" if "ncu_traffic_ratio" in row else ""))
    elif not os.environ.get("SWEEP_NCU_ONLY"):
        import torch
        import paper_1407_6915_b200 as bf
        from synth import gpu as sg
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        elems = int(a.gib * 2 ** 30) // 8
        buf_in = torch.empty(elems, dtype=torch.complex64, device="cuda")
        buf_out = torch.empty_like(buf_in)
        sg.fill_random(buf_in, 1)
        for k in range(a.min, a.max + 1):
            n = 1 << k
            b = elems // n
            x, y = buf_in[: b * n].view(b, n), buf_out[: b * n].view(b, n)
            for d in (-1, 1):
                with bf.Plan(n, b, d) as p:
                    info = p.info()
                    for _ in range(3):
                        p.exec(x, y)
                    best = 1e9
                    for _ in range(10):
                        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        s.record()
                        p.exec(x, y)
                        e.record()
                        e.synchronize()
                        best = min(best, s.elapsed_time(e))
                gbs = 16.0 * n * b / (best * 1e-3) / 1e9
                row = {"log2n": k, "n": n, "dir": d, "batch": b, "variant": info["variant_name"],
                       "ms": best, "alg_GBps": gbs, "frac": gbs / peak, "records_per_s": b / (best * 1e-3)}
                m = ncu.get(k)
                if m and d == -1:
                    tr = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                    row.update(ncu_kernel=m["kernel"][:60], ncu_dram_bytes=tr, ncu_traffic_ratio=tr / (16.0 * n * b),
                               ncu_ms=m.get("gpu__time_duration.sum", 0) * 1e3)
                rows.append(row)
                print(f"N=2^{k:<2} dir={d:+d} {info['variant_name']:>6} batch={b:<8} {best:7.3f} ms "
                      f"{gbs:7.1f} GB/s {gbs / peak:6.1%}" +
                      (f"  ncu DRAM {row['ncu_traffic_ratio']:.3f}x alg" if "ncu_traffic_ratio" in row else ""),
                      flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"config": "config5: sweep 2^8..2^22 fwd+inv, %.0f GiB per N, AUTO plan" % a.gib,
                       "peak_GBps": "MEASURED_PEAKS.json hbm_gbs", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
