"""Summarise an ncu launch list into profiles/ (launch table + per-family DRAM traffic).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file launches.csv python bench.py --steps 1 --warmup 1 ...
    python tools/ncu_summarize.py launches.csv --workload c2_lfr_plm --out profiles/r01_c2_plm_launches_summary.txt

Writes the per-kernel table (total time, share, launches, DRAM bytes per launch) and
merges {workload: {family: {dram_bytes_per_launch, ms_per_launch, launches, share}}}
into profiles/ncu_summary.json, which bench.py reads for roofline.traffic.  ncu's
per-launch times are cold-cache and serialised: only shares are comparable with
the bench's own CUDA-event timings.
"""
import argparse
import collections
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MODE_ARG = {"k_sweep_direct": 1, "k_sweep_warp": 0, "k_sweep_warp_pipe": 0, "k_sweep_block": 0, "k_sweep_thread": 1,
            "k_sweep_cluster": 0, "k_hub_pairs": 0, "k_hub_part": 0, "k_hub_decide": 0}


def family_of(name):
    m = re.search(r"(?:cdk::)?\b(k_\w+)(?:<([^>]*)>)?", name)
    if not m:
        return None
    base, args = m.group(1), m.group(2)
    if base in MODE_ARG and args:
        mode = args.split(",")[MODE_ARG[base]].strip()
        return "plm_move" if mode == "1" else "plp_sweep"
    if base == "k_apply_plm":
        return "plm_apply"
    if base == "k_apply_plp":
        return "plp_apply"
    if base.startswith("k_eng_") or base in ("k_member_count", "k_member_scatter", "k_row_fpre"):
        return "coarsen_or_build"
    return base


def short(name):
    return re.sub(r"\(.*$", "", name.replace("void ", ""))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--cmd", default="")
    ap.add_argument("--runs", type=int, default=1, help="detector runs in the capture (per-step = total / runs)")
    a = ap.parse_args()
    rows = []
    with open(a.csv) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    per = collections.defaultdict(dict)
    for r in rd:
        key = (r["ID"], r["Kernel Name"])
        val = r["Metric Value"].replace(",", "")
        try:
            v = float(val)
        except ValueError:
            continue
        unit = r.get("Metric Unit", "")
        name = r["Metric Name"]
        if name == "gpu__time_duration.sum":
            v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        elif name.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
            v *= scale.get(unit, 1)
        per[key][name] = v
    for (lid, kname), m in per.items():
        rows.append((short(kname), kname, m.get("gpu__time_duration.sum", 0.0),
                     m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)))
    tot_ms = sum(r[2] for r in rows) or 1.0
    by_k = collections.defaultdict(lambda: [0.0, 0, 0.0])
    by_f = collections.defaultdict(lambda: [0.0, 0, 0.0])
    for s, full, ms, b in rows:
        by_k[s][0] += ms
        by_k[s][1] += 1
        by_k[s][2] += b
        fam = family_of(full)
        if fam:
            by_f[fam][0] += ms
            by_f[fam][1] += 1
            by_f[fam][2] += b
    with open(a.out, "w") as f:
        f.write(f"# {a.cmd}\n# ({a.workload}; every launch of the process, cold-cache and serialised by ncu)\n")
        f.write("# total_ms  share  launches  dram_MB/launch  kernel\n")
        for k, (ms, n, b) in sorted(by_k.items(), key=lambda kv: -kv[1][0])[:60]:
            f.write(f"{ms:9.3f} {100 * ms / tot_ms:5.1f}% {n:7d} {b / max(n, 1) / 1e6:12.3f}  {k}\n")
        f.write("\n# families\n")
        for k, (ms, n, b) in sorted(by_f.items(), key=lambda kv: -kv[1][0]):
            f.write(f"{ms:9.3f} {100 * ms / tot_ms:5.1f}% {n:7d} {b / max(n, 1) / 1e6:12.3f}  {k}\n")
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    js = {}
    if os.path.exists(path):
        with open(path) as f:
            js = json.load(f)
    js[a.workload] = {fam: {"dram_bytes_per_launch": b / max(n, 1), "ms_per_launch": ms / max(n, 1),
                            "launches": n, "share": ms / tot_ms, "dram_bytes_per_step": b / max(a.runs, 1),
                            "ms_per_step": ms / max(a.runs, 1), "source": a.cmd or a.csv}
                      for fam, (ms, n, b) in by_f.items()}
    with open(path, "w") as f:
        json.dump(js, f, indent=1, sort_keys=True)
    print(open(a.out).read()[:3000])


if __name__ == "__main__":
    sys.exit(main())
