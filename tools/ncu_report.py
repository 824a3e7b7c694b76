"""Summarise an `ncu --set full` capture (.ncu-rep) into a short text report.

    python tools/ncu_report.py gpurun_out/x.ncu-rep [--top 12] > profiles/x.txt

Per kernel: duration, DRAM bytes and bandwidth, occupancy, L2 hit rate,
occupancy limiters, the non-trivial warp-stall reasons (pc sampling), and the
SASS instructions with the most stall samples (needs -lineinfo).
"""
import argparse
import csv
import io
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__maximum_warps_per_active_cycle_pct",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=12)
    a = ap.parse_args()
    raw = ncu(["-i", a.rep, "--page", "raw", "--csv"])
    rows = list(csv.reader(io.StringIO(raw[raw.index('"ID"'):])))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")]
        print(f"== {name}")
        for k in KEYS:
            if k in h:
                print(f"   {k:70s} {v[h.index(k)]:>14s} {units[h.index(k)]}")
        t = float(v[h.index("gpu__time_duration.sum")].replace(",", ""))
        tu = units[h.index("gpu__time_duration.sum")]
        ts = t * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(tu, 1e-9)
        dram = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            x = float(v[h.index(k)].replace(",", ""))
            dram += x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[h.index(k)], 1)
        print(f"   {'DRAM bandwidth (GB/s)':70s} {dram / ts / 1e9:14.1f}")
        stalls = [(float(v[i].replace(",", "")), w) for i, w in enumerate(h)
                  if "pcsamp_warps_issue_stalled" in w and not w.endswith("not_issued") and v[i]]
        tot = sum(s for s, _ in stalls) or 1.0
        for s, w in sorted(stalls, reverse=True)[:8]:
            if s / tot > 0.02:
                print(f"   stall {w.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * s / tot:5.1f} %")
    src = ncu(["-i", a.rep, "--page", "source", "--csv"])
    if '"Address"' in src:
        srows = list(csv.reader(io.StringIO(src[src.index('"Address"'):])))
        sh = srows[0]
        iS, iW = sh.index("Source"), sh.index("Warp Stall Sampling (All Samples)")
        data = []
        for r in srows[1:]:
            try:
                data.append((int(r[iW]), r[iS].strip()))
            except (ValueError, IndexError):
                pass
        tot = sum(d[0] for d in data) or 1
        print(f"   top SASS by stall samples (of {tot}; first kernel of the capture):")
        for w, s in sorted(data, reverse=True)[:a.top]:
            print(f"   {100 * w / tot:5.1f} %  {s[:80]}")


if __name__ == "__main__":
    main()
