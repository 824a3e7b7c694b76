"""DESIGN.md / README results table from bench JSON lines (profiles/r02_bench).

    python tools/results_table.py profiles/r02_bench"""
import json
import os
import sys

ROWS = [("c3_rmat24_plp", "**C3 PLP (headline)**"), ("c3_rmat24_plm", "C3 PLM"), ("c2_lfr_plm", "C2 PLM"),
        ("c1_planted_plp", "C1 PLP"), ("c1_planted_plm", "C1 PLM"), ("c4_rmat22w_plmr", "C4 PLMR"),
        ("c4_rmat22w_epp", "C4 EPP"), ("c5_rmat28_plp", "C5 PLP (R-MAT s28, one GPU)"),
        ("c5_rmat28_plm", "C5 PLM (R-MAT s28, one GPU)")]


def line(path):
    with open(path) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def main():
    d = sys.argv[1]
    ref_arm = None
    if os.path.exists(os.path.join(d, "c3_ref.json")):
        ref_arm = line(os.path.join(d, "c3_ref.json"))["value"]
    print("| Workload | device ms | device edges/s | e2e ms | e2e edges/s | CPU ref edges/s (16 threads) | device / e2e vs CPU |"
          " Q device / reference (same bytes) | sweep family GB/s (frac of peak) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for key, name in ROWS:
        p = os.path.join(d, key + ".json")
        if not os.path.exists(p):
            continue
        j = line(p)
        q = j.get("quality", {})
        cpu = (j.get("cpu_baseline") or {}).get("value")
        cached = q.get("reference_cached", {})
        refq = None
        for setting in ("parity", "threads"):
            if setting in cached:
                refq = (cached[setting]["modularity"], setting)
                break
        if refq is None and q.get("ref_modularity") is not None:
            refq = (q["ref_modularity"], "live")
        if key == "c3_rmat24_plm" and "threads" in cached:
            cpu = j["config"]["m"] / (cached["threads"]["total_ms"] / 1e3)
            cpu_s = f"{cpu:.2g} (cached, 8 threads)"
        elif cpu:
            cpu_s = f"{cpu:.3g}" + (f" (ref arm {ref_arm:.3g})" if key == "c3_rmat24_plp" and ref_arm else "")
        else:
            cpu_s = "—"
        e2e = j.get("e2e", {})
        ratio = f"{j['value'] / cpu:.0f}× / {e2e['value'] / cpu:.0f}×" if cpu else "—"
        r = j.get("roofline") or {}
        qs = f"{q['modularity']:.6g} / " + (f"{refq[0]:.6g} ({refq[1]})" if refq else "—")
        print(f"| {name} | {j['ms_per_step']:.2f} | {j['value']:.3g} | {e2e.get('ms_per_step', 0):.1f} | "
              f"{e2e.get('value', 0):.3g} | {cpu_s} | {ratio} | {qs} | "
              f"{r.get('achieved', 0):.0f} ({100 * (r.get('frac') or 0):.1f} %) |")


if __name__ == "__main__":
    main()
