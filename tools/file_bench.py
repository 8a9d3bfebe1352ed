"""The file path against a storage roofline (the
on-disk leg; VERDICT r01 "no storage roofline for the file path").

Writes a seeded complex64 file of --gib GiB (records of --n points), measures
the storage with dd (O_DIRECT read, O_DIRECT write, and both at once — the
file pipeline reads and writes concurrently), then runs fft_file on it with
buffered I/O and with O_DIRECT (page cache dropped before each run when the
box allows it), and reports file GB/s = input bytes / wall against the
concurrent dd read / write rates.

  python tools/file_bench.py [--gib 8] [--n 1024] [--dir /tmp/fb] [--json OUT]
"""
import argparse
import json
import os
import re
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1407_6915_b200 as bf  # noqa: E402
from synth import gpu as sg  # noqa: E402


def drop_caches():
    try:
        subprocess.run(["sync"], check=False)
        with open("/proc/sys/vm/drop_caches", "w") as f:
            f.write("3\n")
        return True
    except OSError:
        return False


def dd(args):
    p = subprocess.run(["dd", *args], capture_output=True, text=True)
    m = re.search(r"([\d.]+) s, ([\d.]+) ([GM])B/s", p.stderr)
    if not m:
        return None
    return float(m.group(2)) * (1 if m.group(3) == "G" else 1e-3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=8.0)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--dir", default="/tmp/fb")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    os.makedirs(a.dir, exist_ok=True)
    src, dst, scratch = os.path.join(a.dir, "in.c64"), os.path.join(a.dir, "out.c64"), os.path.join(a.dir, "dd.bin")
    total = int(a.gib * 2 ** 30)
    chunk = 1 << 30
    t = torch.empty(chunk // 8, dtype=torch.complex64, device="cuda")
    with open(src, "wb") as f:
        for off in range(0, total, chunk):
            sg.fill_random(t, 7, first_sample=off // 8)
            f.write(t[: min(chunk, total - off) // 8].cpu().numpy().tobytes())
    del t
    mib = total >> 20
    row = {"file_bytes": total, "n": a.n, "dir": a.dir}
    drop_caches()
    row["dd_read_direct_GBps"] = dd([f"if={src}", "of=/dev/null", "bs=64M", "iflag=direct"])
    row["dd_write_direct_GBps"] = dd(["if=/dev/zero", f"of={scratch}", "bs=64M", f"count={mib // 64}", "oflag=direct"])
    # both at once (what the pipeline does): concurrent read of the input and write of a scratch file
    drop_caches()
    pr = subprocess.Popen(["dd", f"if={src}", "of=/dev/null", "bs=64M", "iflag=direct"], stderr=subprocess.PIPE,
                          text=True)
    pw = subprocess.Popen(["dd", "if=/dev/zero", f"of={scratch}", "bs=64M", f"count={mib // 64}", "oflag=direct"],
                          stderr=subprocess.PIPE, text=True)
    er, ew = pr.communicate()[1], pw.communicate()[1]
    gr = re.search(r"([\d.]+) ([GM])B/s", er)
    gw = re.search(r"([\d.]+) ([GM])B/s", ew)
    row["dd_concurrent_read_GBps"] = float(gr.group(1)) * (1 if gr.group(2) == "G" else 1e-3) if gr else None
    row["dd_concurrent_write_GBps"] = float(gw.group(1)) * (1 if gw.group(2) == "G" else 1e-3) if gw else None
    os.unlink(scratch)
    for direct in (False, True):
        for rep in range(2):
            dropped = drop_caches()
            t0 = time.perf_counter()
            st = bf.fft_file(src, dst, a.n, 1, options=bf.StreamOptions(direct_io=direct, io_threads=8))
            wall = time.perf_counter() - t0
            key = f"fft_file_{'direct' if direct else 'buffered'}_{rep}"
            row[key] = {"GBps_in": total / wall / 1e9, "wall_s": wall, "cache_dropped": dropped,
                        "direct_io_used": st["direct_io"], "read_s": st["read_s"], "write_s": st["write_s"],
                        "h2d_s": st["h2d_s"], "fft_s": st["fft_s"], "d2h_s": st["d2h_s"]}
            print(key, json.dumps(row[key]), flush=True)
            os.unlink(dst)
    best = max(v["GBps_in"] for k, v in row.items() if k.startswith("fft_file_"))
    roof = min(x for x in (row["dd_concurrent_read_GBps"], row["dd_concurrent_write_GBps"]) if x)
    row["best_fft_file_GBps"] = best
    row["storage_roofline_GBps"] = roof
    row["frac_of_storage_roofline"] = best / roof if roof else None
    os.unlink(src)
    print(json.dumps({k: v for k, v in row.items() if not k.startswith("fft_file_")}))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(row, f, indent=1)


if __name__ == "__main__":
    main()
