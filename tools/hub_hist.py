import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1304_4453_b200 as P, bench
ctx = P.Context(0)
g = bench.make_device_graph(P, ctx, bench.WORKLOADS['c3_rmat24_plm'])
for level in range(2):
    deg = np.diff(g.csr()['off'])
    edges = [4096, 8192, 16384, 32768, 65536, 131072, 262144, 1 << 30]
    lo = 4096
    out = []
    for hi in edges[1:]:
        sel = (deg > lo) & (deg <= hi)
        out.append((lo, hi, int(sel.sum()), int(deg[sel].sum())))
        lo = hi
    print('level', level, 'entries', int(deg.sum()), out, flush=True)
    z, _ = P.move_phase(g, np.arange(g.node_count(), dtype=np.int32), P.LouvainConfig())
    zc, _ = P.compacted(z, ctx=ctx)
    g, _ = P.coarsen(g, zc)
