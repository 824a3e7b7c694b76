"""Quality / time tradeoff of the device update order.

    python tools/param_sweep.py [--ref]

Runs PLM on the bench graphs with bucket counts, singleton guard and
move-phase stop tolerance varied, printing modularity, time and passes; with
--ref also the reference's PLM modularity (oracle/_ref, all host threads).
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1304_4453_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--graphs", default="c1,c2,r20,r20w")
    ap.add_argument("--variants", default=None,
                    help="';'-separated LouvainConfig overrides, e.g. 'move_tol=1e-3;move_tol=1e-2,prune=2'")
    a = ap.parse_args()
    ctx = P.Context(0)
    graphs = {}
    names = a.graphs.split(",")
    if "c1" in names:
        graphs["c1"] = P.generate_planted(100000, 1000, 0.1, 2 / 99900, 1, ctx=ctx)[0]
    if "c2" in names:
        graphs["c2"] = P.generate_lfr(seed=1, ctx=ctx, **bench.LFR_C2)[0]
    if "r20" in names:
        graphs["r20"] = P.generate_rmat(20, 16, weighted=False, seed=1, ctx=ctx)
    if "r20w" in names:
        graphs["r20w"] = P.generate_rmat(20, 16, weighted=True, seed=1, ctx=ctx)
    variants = []
    for stall in (0.0, 0.95, 0.9):
        for tol in (0.0, 1e-3):
            variants.append(dict(buckets=4, move_tol=tol, move_stall=stall, singleton_guard=True))
    variants.append(dict(buckets=8, move_tol=1e-3, move_stall=0.95, singleton_guard=True))
    if a.variants:
        variants = []
        for spec in a.variants.split(";"):
            d = {}
            for kv in filter(None, spec.split(",")):
                k, v = kv.split("=")
                d[k] = type(getattr(P.LouvainConfig(), k))(eval(v))
            variants.append(d)
    for name, g in graphs.items():
        for v in variants:
            for refine in (False,):
                cfg = P.LouvainConfig(refine=refine, **v)
                P.run_louvain(g, cfg)
                ts = []
                for _ in range(3):
                    z, rep = P.run_louvain(g, cfg)
                    ts.append(rep.total_ms)
                print(f"{name} m={g.edge_count()} {v} refine={refine} Q={rep.modularity:.6f} k={rep.community_count} "
                      f"ms={min(ts):.2f} passes={[l['passes'] for l in rep.levels]}", flush=True)
        if a.ref:
            from oracle import oracle as O
            c = g.csr()
            og = O.from_csr(g.node_count(), c["off"], c["col"], None if c["w"] is None else c["w"].astype("float64"))
            rg = O.RefGraph.from_csr(og)
            t0 = time.time()
            zr, rr = rg.run_louvain(refine=False, workers=bench.cpu_threads())
            print(f"{name} REF plm Q={rr['modularity']:.6f} k={rr['community_count']} ms={rr['total_ms']:.1f} "
                  f"wall={time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
