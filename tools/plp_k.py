"""PLP bucket-count sweep: time, iterations and modularity per K (one B200).

    python tools/plp_k.py [--workload c3_rmat24_plp] [--ks 2 3 4 6 8]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1304_4453_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_rmat24_plp")
    ap.add_argument("--ks", type=int, nargs="+", default=[2, 3, 4, 6, 8])
    a = ap.parse_args()
    ctx = P.Context(0)
    g = bench.make_device_graph(P, ctx, bench.WORKLOADS[a.workload])
    for k in a.ks:
        best = None
        for _ in range(3):
            z, rep = P.run_plp(g, P.PlpConfig(buckets=k))
            best = rep if best is None or rep.total_ms < best.total_ms else best
        print(f"{a.workload} K={k}: {best.total_ms:.3f} ms, {len(best.iterations)} iterations, "
              f"Q={best.modularity:.6f}, k={best.community_count}", flush=True)


if __name__ == "__main__":
    main()
