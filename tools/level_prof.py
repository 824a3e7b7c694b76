"""Per-level anatomy of a Louvain run (which kernels a coarse level spends on).

    python tools/level_prof.py [--workload c2_lfr_plm] [--levels 3]

Rebuilds the level graphs of a PLM run through the public API (move phase ->
compact -> coarsen) and, for each level, prints its shape (n, entries,
degree tiers), the un-profiled move-phase time and the per-family kernel
times of a profiled repeat.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1304_4453_b200 as P  # noqa: E402

TIERS = [(8, "g8"), (16, "g16"), (32, "g32"), (256, "warp"), (1024, "block"), (4096, "block2"), (8192, "block3"),
         (65536, "cluster"),
         (1 << 62, "hub")]


def tiers(g):
    deg = np.diff(g.csr()["off"])
    out, lo = {}, 0
    for hi, name in TIERS:
        sel = (deg > lo) & (deg <= hi)
        if sel.any():
            out[name] = (int(sel.sum()), int(deg[sel].sum()))
        lo = hi
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2_lfr_plm", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--start", type=int, default=0, help="levels below this only run once (ncu --launch-skip)")
    ap.add_argument("--buckets", type=int, default=4)
    a = ap.parse_args()
    wl = bench.WORKLOADS[a.workload]
    ctx = P.Context(0)
    g = bench.make_device_graph(P, ctx, wl)
    cfg = P.LouvainConfig(buckets=a.buckets)
    for level in range(a.levels):
        # louvain_recurse prunes only the input graph's move phases
        cfg = P.LouvainConfig(buckets=a.buckets, prune=1 if level == 0 else 0)
        n = g.node_count()
        z0 = np.arange(n, dtype=np.int32)
        if level < a.start:
            z, changed = P.move_phase(g, z0.copy(), cfg)
            zc, _ = P.compacted(z, ctx=ctx)
            g, _ = P.coarsen(g, zc)
            continue
        P.move_phase(g, z0.copy(), cfg)  # warm (bins, graphs)
        ctx.synchronize()
        t0 = time.perf_counter()
        z, changed = P.move_phase(g, z0.copy(), cfg)
        ms = 1e3 * (time.perf_counter() - t0)
        ctx.reset_stats()
        ctx.set_profiling(True)
        P.move_phase(g, z0.copy(), cfg)
        ctx.set_profiling(False)
        st = ctx.kernel_stats()
        fams = sorted(((k, v["total_ms"], v["launches"]) for k, v in st.items() if k not in ("plm_move",)),
                      key=lambda x: -x[1])
        print(f"level {level}: n={n} entries={g.entries} tiers={tiers(g)} move_wall_ms={ms:.2f}")
        for k, t, l in fams[:12]:
            print(f"    {k:18s} {t:8.3f} ms  {l:5d} launches  {1e3 * t / max(l, 1):8.1f} us/launch")
        if not changed:
            break
        zc, _ = P.compacted(z, ctx=ctx)
        g, _ = P.coarsen(g, zc)


if __name__ == "__main__":
    main()
