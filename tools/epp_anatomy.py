import sys; sys.path.insert(0,'/root/repo')
import paper_1304_4453_b200 as P, bench
ctx=P.Context(0)
g=bench.make_device_graph(P, ctx, bench.WORKLOADS['c4_rmat22w_epp'])
for i in range(3):
    z, rep = P.run_epp(g, P.EnsembleConfig())
    print(rep.total_ms, rep.base_ms, rep.combine_ms, rep.coarsen_ms, rep.final_ms, rep.community_count, rep.modularity)
z, rep = P.run_plp(g, P.PlpConfig(randomize_order=True))
print('plp', rep.total_ms, len(rep.iterations), [it['updated'] for it in rep.iterations][:12])
