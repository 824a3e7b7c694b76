"""Stress the C5-sized paths on one GPU: R-MAT at a large scale through PLP,
PLM, PLMR (refinement re-bins graphs that released their tier lists) and EPP
(bases serial above 2^31 entries), printing time and quality per detector."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_1304_4453_b200 as P  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
    algos = sys.argv[2].split(",") if len(sys.argv) > 2 else ["plp", "plm", "plmr", "epp"]
    ctx = P.default_context()
    t0 = time.time()
    g = P.generate_rmat(scale, 16, seed=1, ctx=ctx)
    print(json.dumps({"scale": scale, "build_s": round(time.time() - t0, 2), "D": g.entries}), flush=True)
    for a in algos:
        t0 = time.time()
        if a == "plp":
            z, rep = P.run_plp(g, P.PlpConfig())
        elif a == "plm":
            z, rep = P.run_plm(g, P.LouvainConfig())
        elif a == "plmr":
            z, rep = P.run_plmr(g, P.LouvainConfig())
        else:
            z, rep = P.run_epp(g, P.EnsembleConfig(ensemble_size=2))
        print(json.dumps({"algo": a, "wall_s": round(time.time() - t0, 2), "modularity": rep.modularity,
                          "communities": rep.community_count}), flush=True)


if __name__ == "__main__":
    main()
