"""Probe: build the R-MAT graph at a given scale with the chunked builder and
run PLP / PLM on it, printing build time, size, device memory and the
detector times (SURVEY.md §8(d) C3 / C5 sizes on one GPU)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_1304_4453_b200 as P  # noqa: E402


def mem():
    import torch
    f, t = torch.cuda.mem_get_info()
    return round((t - f) / 2**30, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--algos", default="plm")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.out:
        sys.stdout = open(args.out, "w", buffering=1)
    ctx = P.default_context()
    t0 = time.time()
    g = P.generate_rmat(args.scale, args.ef, seed=1, ctx=ctx)
    ctx.synchronize() if hasattr(ctx, "synchronize") else None
    out = {"scale": args.scale, "build_s": round(time.time() - t0, 2), "n": g.node_count(), "m": g.edge_count(),
           "D": g.entries, "max_degree": g.max_degree, "isolated": g.isolated, "mem_gib_after_build": mem()}
    print(json.dumps(out), flush=True)
    for a in args.algos.split(","):
        t0 = time.time()
        if a == "plp":
            z, rep = P.run_plp(g, P.PlpConfig())
        else:
            z, rep = P.run_plm(g, P.LouvainConfig())
        dt = time.time() - t0
        print(json.dumps({"algo": a, "wall_s": round(dt, 3), "total_ms": rep.total_ms, "modularity": rep.modularity,
                          "communities": rep.community_count, "edges_per_s": g.edge_count() / (rep.total_ms / 1e3),
                          "mem_gib": mem()}), flush=True)
        for lv in getattr(rep, "levels", []) or []:
            print(json.dumps(lv), flush=True)


if __name__ == "__main__":
    main()
