"""Single-workload driver for ncu captures (profiles/README.md).

    python tools/prof_run.py [--workload c2_lfr_plm] [--runs 2]

Generates the bench workload on cuda:0 and runs the detector `runs` times
(the first is a warm-up).  Prints one line with the per-level report.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1304_4453_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2_lfr_plm", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--set", action="append", default=[], help="LouvainConfig field=value (PLM/PLMR)")
    ap.add_argument("--families", action="store_true", help="per-family kernel times of one profiled run")
    a = ap.parse_args()
    over = {}
    for kv in a.set:
        k, v = kv.split("=")
        over[k] = type(getattr(P.LouvainConfig(), k))(eval(v))
    wl = bench.WORKLOADS[a.workload]
    ctx = P.Context(0)
    g = bench.make_device_graph(P, ctx, wl)
    for i in range(a.runs):
        if over and wl["algo"] in ("plm", "plmr"):
            z, rep = P.run_louvain(g, P.LouvainConfig(refine=wl["algo"] == "plmr", **over))
        else:
            z, rep = bench.run_device(P, g, wl["algo"], None, report=True)
        print(a.workload, "run", i, "m", g.edge_count(), "Q", round(rep.modularity, 6), "k", rep.community_count,
              "ms", round(rep.total_ms, 3),
              "levels", [(l["nodes"], l["passes"], round(l["move_ms"], 2), round(l["coarsen_ms"], 2))
                         for l in rep.levels], "iters", [(it["updated"], round(it["ms"], 3)) for it in rep.iterations],
              flush=True)
    if a.families:
        ctx.reset_stats()
        ctx.set_profiling(True)
        bench.run_device(P, g, wl["algo"], None, report=False)
        ctx.set_profiling(False)
        st = ctx.kernel_stats()
        for k, v in sorted(st.items(), key=lambda kv: -kv[1]["total_ms"])[:30]:
            print(f"  {k:28s} {v['total_ms']:9.3f} ms {v['launches']:6d} launches")


if __name__ == "__main__":
    main()
