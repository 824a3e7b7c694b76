"""Share of each degree tier's entries whose label equals the node's own
label after PLP iterations 1..3 (the own-label bypass), on an
R-MAT graph through the C port of the device order (runs on CPU).

    python tools/own_label_probe.py [--scale 20]"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

TIERS = ((1, 8, "g8"), (9, 32, "g16-32"), (33, 256, "warp"), (257, 8192, "block"), (8193, 1 << 62, "cluster/hub"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    a = ap.parse_args()
    g = O.generate_rmat(a.scale, 16, 0.57, 0.19, 0.19, seed=1)
    n = len(g.off) - 1
    deg = np.diff(g.off)
    rows = np.repeat(np.arange(n), deg)
    for it in (1, 2, 3):
        z, _ = O.plp_bucketed(g, max_iterations=it)
        z = np.asarray(z)
        own = np.bincount(rows, weights=(z[g.col] == z[rows]), minlength=n)
        for lo, hi, name in TIERS:
            m = (deg >= lo) & (deg <= hi)
            ent = deg[m].sum()
            maj = 2 * own[m] > deg[m]
            print(f"iteration {it} {name:12s} nodes {int(m.sum()):9d} entries {int(ent):10d} "
                  f"own-label entries {own[m].sum() / max(ent, 1):.3f} own-majority nodes {maj.mean():.3f}")


if __name__ == "__main__":
    main()
