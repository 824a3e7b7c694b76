"""Per-iteration anatomy of a PLP run: each tier family's kernel time in
iteration i, from serialised profiled runs capped at i and i-1 iterations
(the run is deterministic, so the difference is iteration i alone).

    python tools/iter_prof.py [--workload c3_rmat24_plp] [--iters 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1304_4453_b200 as P  # noqa: E402


def fams(ctx, g, cap):
    ctx.reset_stats()
    ctx.set_profiling(True)
    lab, rep = P.run_plp(g, P.PlpConfig(max_iterations=cap), report=True)
    ctx.set_profiling(False)
    return {k: v["total_ms"] for k, v in ctx.kernel_stats().items()}, rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_rmat24_plp")
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    ctx = P.Context(0)
    g = bench.make_device_graph(P, ctx, bench.WORKLOADS[a.workload])
    P.run_plp(g, P.PlpConfig())  # warm-up (tier lists, graphs)
    prev = {}
    for it in range(1, a.iters + 1):
        cur, rep = fams(ctx, g, it)
        diff = {k: cur.get(k, 0.0) - prev.get(k, 0.0) for k in cur}
        top = sorted(((v, k) for k, v in diff.items() if v > 0.005), reverse=True)
        upd = rep.iterations[-1]["updated"] if rep.iterations else 0
        print(f"iter {it} updated {upd} total {sum(v for v, _ in top):.3f} ms: "
              + " ".join(f"{k}={v:.3f}" for v, k in top[:14]), flush=True)
        prev = cur


if __name__ == "__main__":
    main()
