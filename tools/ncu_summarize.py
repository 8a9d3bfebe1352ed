"""Summarise an ncu --set full report (.ncu-rep) as markdown: key throughput
metrics, DRAM bytes vs algorithmic bytes, warp-stall breakdown and the top
stalled SASS lines.  Usage: python tools/ncu_summarize.py rep.ncu-rep [alg_bytes]"""
import csv
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return {h: (v, u) for h, u, v in zip(r[0], r[1], r[2])}


def source(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[1], r[2:]


def main():
    rep = sys.argv[1]
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    m = raw(rep)
    print(f"# ncu summary: `{rep.split('/')[-1]}`\n")
    print(f"Kernel: `{m.get('Kernel Name', ('?',))[0]}`\n")
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__m_l1tex2xbar_write_bytes_mem_dshared.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__cluster_max_active", "sm__cycles_elapsed.avg.per_second"]
    print("| metric | value | unit |\n|---|---|---|")
    for k in keys:
        if k in m:
            print(f"| {k} | {m[k][0]} | {m[k][1]} |")
    try:
        rd = float(m["dram__bytes_read.sum"][0].replace(",", ""))
        wr = float(m["dram__bytes_write.sum"][0].replace(",", ""))
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
        rd *= scale.get(m["dram__bytes_read.sum"][1], 1)
        wr *= scale.get(m["dram__bytes_write.sum"][1], 1)
        print(f"\nDRAM traffic per launch: {rd + wr:.4g} B", end="")
        if alg:
            print(f" = {(rd + wr) / alg:.3f} x algorithmic ({alg:.4g} B)")
        else:
            print()
    except (KeyError, ValueError):
        pass
    hdr, data = source(rep)
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[i_s] or 0) for r in data) or 1
    agg = {c: sum(float(r[hdr.index(c)] or 0) for r in data) for c in cols}
    print("\nWarp-stall breakdown (share of samples):\n")
    print(", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v / tot > 0.005))
    print("\nTop stalled SASS:\n\n```")
    for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:12]:
        print(f"{float(r[i_s]) / tot:6.1%}  {r[1][:90]}")
    print("```")


if __name__ == "__main__":
    main()
