"""A/B timing of one workload: median device time of complete runs (L2
flushed before each, CUDA events on the library stream) and the per-family
kernel times of one serialised profiled run.  Environment knobs (CD_*) are
read by the library once per process, so each variant is its own process:

    CD_WARP_PIPE=0 python tools/ab_time.py --workload c2_lfr_plm --runs 7
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1304_4453_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", action="append", default=[])
    ap.add_argument("--runs", type=int, default=7)
    ap.add_argument("--tag", default=os.environ.get("AB_TAG", ""))
    ap.add_argument("--families", type=int, default=12)
    a = ap.parse_args()
    import torch

    ctx = P.Context(0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
    stream = torch.cuda.ExternalStream(ctx.stream, device="cuda:0")
    for name in a.workload or ["c2_lfr_plm"]:
        wl = bench.WORKLOADS[name]
        g = bench.make_device_graph(P, ctx, wl)
        out = torch.empty(max(g.node_count(), 1), dtype=torch.int32, device="cuda:0")
        for _ in range(2):
            bench.run_device(P, g, wl["algo"], out, report=False)
        ts = []
        for _ in range(a.runs):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            bench.run_device(P, g, wl["algo"], out, report=False)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        z, rep = bench.run_device(P, g, wl["algo"], None, report=True)
        print(f"AB {a.tag} {name} median_ms {statistics.median(ts):.3f} min_ms {min(ts):.3f} max_ms {max(ts):.3f} "
              f"Q {rep.modularity:.6f} k {rep.community_count}", flush=True)
        ctx.reset_stats()
        ctx.set_profiling(True)
        bench.run_device(P, g, wl["algo"], None, report=False)
        ctx.set_profiling(False)
        st = ctx.kernel_stats()
        for k, v in sorted(st.items(), key=lambda kv: -kv[1]["total_ms"])[:a.families]:
            print(f"   {a.tag} {name} {k:26s} {v['total_ms']:9.3f} ms {v['launches']:6d}", flush=True)
        del g, out


if __name__ == "__main__":
    main()
