"""Row-engine workload of C3's level-0 contraction: source lengths (sum of
member degrees) and distinct lengths (coarse degrees) of the coarse rows.

    python tools/coarse_rows.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1304_4453_b200 as P  # noqa: E402


def main():
    ctx = P.Context(0)
    g = bench.make_device_graph(P, ctx, bench.WORKLOADS["c3_rmat24_plm"])
    n = g.node_count()
    z, _ = P.move_phase(g, np.arange(n, dtype=np.int32), P.LouvainConfig())
    zc, k = P.compacted(z)
    c = g.csr()
    deg = np.diff(c["off"])
    F = np.bincount(zc, weights=deg, minlength=k).astype(np.int64)
    cg, _ = P.coarsen(g, zc)
    cd = np.diff(cg.csr()["off"])
    order = np.argsort(-F)
    print(f"n={n} k={k} D={g.entries} coarse D={cg.entries}")
    for lo, hi in [(0, 32), (33, 256), (257, 4096), (4097, 1 << 62)]:
        m = (F >= lo) & (F <= hi)
        print(f"F in [{lo},{hi}]: rows {int(m.sum())} entries {int(F[m].sum())} distinct {int(cd[m].sum())}")
    for r in order[:12]:
        print(f"  row {r}: F={F[r]} distinct={cd[r]} members={int((zc == r).sum())}")


if __name__ == "__main__":
    main()
    sys.stdout.flush()
    os._exit(0)
