"""Warp-tier phase anatomy (debug build with -DCD_PHASE_TIMING).

    COMMDET_CUDA_LIB=build/libphase.so python tools/phase_prof.py

Average clock64 cycles per node of the warp tier's phases (lane 0 view):
0 row bounds, 1 clear + row loads issued, 2 label gathers, 3 tally inserts,
4 candidate scan, 5 decision + queue, at level 0 and level 1 of C2 PLM.
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1304_4453_b200 as P  # noqa: E402


def main():
    L = P.load_library()
    fn = L.cd_debug_phase
    fn.argtypes = [C.c_void_p]
    buf = np.zeros(16, np.uint64)
    ctx = P.Context(0)
    g = bench.make_device_graph(P, ctx, bench.WORKLOADS["c2_lfr_plm"])
    cfg = P.LouvainConfig()
    for level in range(3):
        z0 = np.arange(g.node_count(), dtype=np.int32)
        fn(buf.ctypes.data)
        z, _ = P.move_phase(g, z0, cfg)
        fn(buf.ctypes.data)
        nodes = max(int(buf[8]), 1)
        ph = [int(x) / nodes for x in buf[:6]]
        print(f"level {level}: warp-tier nodes {nodes} avg deg {int(buf[9]) / nodes:.1f} cycles/node "
              + " ".join(f"{x:.0f}" for x in ph) + f" total {sum(ph):.0f}")
        zc, _ = P.compacted(z, ctx=ctx)
        g, _ = P.coarsen(g, zc)


if __name__ == "__main__":
    main()
