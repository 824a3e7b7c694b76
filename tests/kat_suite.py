"""Known-answer tests of the reference's unit suite (T/test_*.cpp), written
once against a small Backend protocol and run twice:

  * tests/test_oracle_kat.py  -- the C oracle (CPU),
  * tests/test_gpu_kat.py     -- the product library on cuda:0 (GPU).

Each test cites the reference test it re-expresses (Catch2 is absent here).
Graph instances mirror T/oracles.hpp:131-199 with numpy's PCG64; weights are
integers so fp32 device storage is exact.
"""
import numpy as np
import pytest

from conftest import BARBELL, TRIANGLES, TWO_TRIANGLES, rand_edges, refines, same_relation


class OracleBackend:
    def __init__(self, O):
        self.O = O
        self.InputError = O.OracleInputError
        self.InvalidArgument = O.OracleInvalidArgument
        self.DomainError = O.OracleDomainError
        self.OutOfRange = O.OracleOutOfRange

    def graph(self, n, edges, merge=False):
        return self.O.from_edges(n, edges, merge)

    def arrays(self, n, eu, ev, ew):
        return self.O.from_arrays(n, eu, ev, ew)

    def csr(self, g):
        return dict(n=g.n, off=g.off, col=g.col, w=g.w, vol=g.vol, loop=g.loop, m=g.m, total=g.total)

    def modularity(self, g, z, gamma=1.0):
        return self.O.modularity(g, z, gamma, ub=int(np.max(z)) + 1 if len(z) else 1)

    def coverage(self, g, z):
        return self.O.coverage(g, z)

    def dominant_label(self, g, z, u):
        return self.O.dominant_label(g, z, u)

    def is_stable(self, g, z):
        return self.O.is_stable(g, z)

    def plp(self, g, theta=-1, max_iterations=100, seed=1, initial=None):
        if g.total == 0.0 and g.n and initial is None:
            pass
        return self.O.plp_bucketed(g, theta=theta, max_iterations=max_iterations, seed=seed, initial=initial)

    def plm(self, g, refine=False, gamma=1.0, seed=1):
        if g.total == 0.0:
            raise self.DomainError("Louvain requires positive total edge weight")
        z, k, lv = self.O.louvain_bucketed(g, refine=refine, gamma=gamma, seed=seed)
        return z, self.O.modularity(g, z, gamma)

    def epp(self, g, b=4, seed=1):
        z, k = self.O.epp_bucketed(g, ensemble_size=b, seed=seed)
        return z, self.O.modularity(g, z)

    def coarsen(self, g, z):
        return self.O.coarsen(g, z), np.asarray(z, np.int32)

    def prolong(self, zc, pi):
        return self.O.prolong(zc, pi)

    def compact(self, z):
        return self.O.compact(z)

    def combine(self, sols):
        return self.O.combine_hashed(sols)

    def planted(self, n, k, pin, pout, seed):
        return self.O.generate_planted(n, k, pin, pout, seed)


class DeviceBackend:
    def __init__(self, P):
        self.P = P
        self.InputError = P.InputError
        self.InvalidArgument = P.InvalidArgument
        self.DomainError = P.DomainError
        self.OutOfRange = P.OutOfRange

    def graph(self, n, edges, merge=False):
        return self.P.Graph.from_edges(n, edges, merge_duplicates=merge)

    def arrays(self, n, eu, ev, ew):
        return self.P.Graph.from_edges(n, (eu, ev, ew.astype(np.float32)))

    def csr(self, g):
        c = g.csr()
        w = c["w"].astype(np.float64) if c["w"] is not None else np.ones(len(c["col"]))
        return dict(n=g.node_count(), off=c["off"], col=c["col"], w=w, vol=c["vol"], loop=c["loop"],
                    m=g.edge_count(), total=g.total_edge_weight())

    def modularity(self, g, z, gamma=1.0):
        return self.P.modularity(g, z, gamma)

    def coverage(self, g, z):
        return self.P.coverage(g, z)

    def dominant_label(self, g, z, u):
        return self.P.dominant_label(g, z, u)

    def is_stable(self, g, z):
        return self.P.is_stable(g, z)

    def plp(self, g, theta=-1, max_iterations=100, seed=1, initial=None):
        z, rep = self.P.run_plp(g, self.P.PlpConfig(theta=theta, max_iterations=max_iterations, seed=seed),
                                initial=initial)
        return z, np.array([it["updated"] for it in rep.iterations], np.int64)

    def plm(self, g, refine=False, gamma=1.0, seed=1):
        z, rep = self.P.run_louvain(g, self.P.LouvainConfig(gamma=gamma, refine=refine, seed=seed))
        return z, rep.modularity

    def epp(self, g, b=4, seed=1):
        z, rep = self.P.run_epp(g, self.P.EnsembleConfig(ensemble_size=b, seed=seed))
        return z, rep.modularity

    def coarsen(self, g, z):
        return self.P.coarsen(g, z)

    def prolong(self, zc, pi):
        return self.P.prolong(zc, pi)

    def compact(self, z):
        return self.P.compacted(z)

    def combine(self, sols):
        return self.P.combine_hashed(sols)

    def planted(self, n, k, pin, pout, seed):
        return self.P.generate_planted(n, k, pin, pout, seed)


# ---------------------------------------------------------------------------
# T/test_graph.cpp
# ---------------------------------------------------------------------------
def kat_graph_counts(B):
    g = B.graph(0, [])
    c = B.csr(g)
    assert c["n"] == 0 and c["m"] == 0 and c["total"] == 0.0  # empty graph (:12-17)
    c = B.csr(B.graph(6, BARBELL))  # barbell counts (:19-26)
    assert c["n"] == 6 and c["m"] == 7 and c["total"] == 7.0
    assert c["vol"][2] == 3.0 and c["off"][3] - c["off"][2] == 3
    c = B.csr(B.graph(1, [(0, 0, 2.0)]))  # self-loop (:28-33)
    assert c["total"] == 2.0 and c["vol"][0] == 4.0 and c["loop"][0] == 2.0
    c = B.csr(B.graph(3, [(0, 1, 1)]))  # isolated node (:35-39)
    assert c["vol"][2] == 0.0 and c["off"][3] - c["off"][2] == 0


def kat_graph_errors(B):
    # build rejects bad edges (T/test_graph.cpp:41-47)
    for n, edges in [(2, [(0, 2, 1)]), (2, [(0, 1, 0.0)]), (2, [(0, 1, -1.0)]), (2, [(0, 1, 1), (1, 0, 1)]),
                     (2, [(0, 1, 1), (0, 1, 2)])]:
        with pytest.raises(B.InputError):
            B.graph(n, edges)
    c = B.csr(B.graph(2, [(0, 1, 1), (1, 0, 1)], merge=True))  # merge (:49-54)
    assert c["m"] == 1 and c["total"] == 2.0 and c["vol"][0] == 2.0
    c = B.csr(B.graph(2, [(0, 1), (1, 0)], merge=True))  # unweighted input: merged weight 2
    assert c["m"] == 1 and c["total"] == 2.0 and c["vol"][0] == 2.0


def kat_graph_random_invariants(B):
    rng = np.random.default_rng(42)
    for i in range(30):  # handshake (:78-86) and symmetry (:88-102)
        n = 2 + i % 20
        eu, ev, ew = rand_edges(rng, n, 0.3, "int" if i % 2 == 0 else "dyadic", loop_p=0.2)
        c = B.csr(B.arrays(n, eu, ev, ew))
        assert np.sum(c["vol"]) == pytest.approx(2.0 * c["total"], rel=1e-12)
        for u in range(n):
            for j in range(c["off"][u], c["off"][u + 1]):
                v = c["col"][j]
                if j > c["off"][u]:
                    assert c["col"][j - 1] < v  # rows strictly ascending
                if v != u:
                    row = c["col"][c["off"][v]:c["off"][v + 1]]
                    k = np.searchsorted(row, u)
                    assert row[k] == u and c["w"][c["off"][v] + k] == c["w"][j]


# ---------------------------------------------------------------------------
# T/test_quality.cpp
# ---------------------------------------------------------------------------
def kat_modularity_known(B):
    bar = B.graph(6, BARBELL)
    assert B.modularity(bar, np.zeros(6, np.int32)) == pytest.approx(0.0, abs=1e-15)  # (:35-43)
    assert B.modularity(bar, TRIANGLES) == pytest.approx(5.0 / 14.0, abs=1e-15)
    assert B.modularity(B.graph(6, TWO_TRIANGLES), TRIANGLES) == pytest.approx(0.5, abs=1e-15)
    assert B.coverage(bar, TRIANGLES) == pytest.approx(6.0 / 7.0, abs=1e-15)  # (:16-21)
    assert B.coverage(bar, np.zeros(6, np.int32)) == 1.0
    assert B.coverage(bar, np.arange(6, dtype=np.int32)) == 0.0
    empty = B.graph(4, [])
    assert B.coverage(empty, np.arange(4, dtype=np.int32)) == 0.0  # (:23-28)
    with pytest.raises(B.DomainError):  # (:45-48)
        B.modularity(empty, np.arange(4, dtype=np.int32))


def kat_modularity_identity(B):
    rng = np.random.default_rng(5)  # Q = coverage - penalty (:74-87)
    for i in range(30):
        n = 4 + i % 10
        eu, ev, ew = rand_edges(rng, n, 0.5)
        g = B.graph(n, list(zip(eu.tolist(), ev.tolist(), ew.tolist())))
        c = B.csr(g)
        z = rng.integers(0, 3, n).astype(np.int32)
        vol = np.zeros(3)
        np.add.at(vol, z, c["vol"])
        pen = float(np.sum(vol * vol) / (4.0 * c["total"] ** 2))
        q = B.modularity(g, z)
        assert q == pytest.approx(B.coverage(g, z) - pen, abs=1e-9)
        assert -1.0 < q <= 1.0  # bounds (:89-98)


# ---------------------------------------------------------------------------
# T/test_plp.cpp
# ---------------------------------------------------------------------------
def kat_dominant_label(B):
    g = B.graph(6, [(0, 1, 5), (0, 2, 1), (0, 3, 1), (0, 4, 1), (0, 5, 1)])
    assert B.dominant_label(g, np.array([0, 1, 7, 7, 7, 7], np.int32), 0) == 1  # 5 > 4 (:21-28)
    h = B.graph(3, [(0, 1, 3), (0, 2, 2)])
    assert B.dominant_label(h, np.array([9, 1, 2], np.int32), 0) == 1  # (:29-34)
    assert B.dominant_label(B.graph(6, BARBELL), np.arange(6, dtype=np.int32), 0) == 1  # tie (:37-41)
    with pytest.raises(B.InvalidArgument):  # isolated (:43-46)
        B.dominant_label(B.graph(2, []), np.arange(2, dtype=np.int32), 0)
    assert B.dominant_label(B.graph(2, [(0, 0, 3), (0, 1, 1)]), np.arange(2, dtype=np.int32), 0) == 0  # (:48-52)


def kat_plp_runs(B):
    g = B.graph(6, TWO_TRIANGLES)
    z, trace = B.plp(g, theta=0)  # (:54-60)
    assert len(set(z.tolist())) == 2
    assert B.modularity(g, B.compact(z)[0]) == pytest.approx(0.5, abs=1e-12)
    assert len(trace) >= 1
    e = B.graph(5, [])
    z, trace = B.plp(e, theta=1)  # edgeless (:62-68)
    assert np.array_equal(z, np.arange(5)) and list(trace) == [0]
    bar = B.graph(6, BARBELL)
    z, _ = B.plp(bar, theta=0)  # barbell fixed point (:70-75)
    assert B.is_stable(bar, z) and B.coverage(bar, z) >= 6.0 / 7.0
    assert B.is_stable(g, TRIANGLES)  # (:77-81)
    assert not B.is_stable(g, np.arange(6, dtype=np.int32))
    z, trace = B.plp(g, theta=0, initial=TRIANGLES)  # initial partition honoured (:129-134)
    assert same_relation(z, TRIANGLES) and trace[0] == 0


def kat_plp_random(B):
    rng = np.random.default_rng(31)
    for i in range(20):  # theta = 0 => stable (:83-90)
        n = 5 + i
        eu, ev, ew = rand_edges(rng, n, 0.3, "unit", loop_p=0.1)
        g = B.arrays(n, eu, ev, ew)
        z, trace = B.plp(g, theta=0)
        assert B.is_stable(g, z)
        assert np.all(z < n)  # labels conserved (:117-127)
    rng = np.random.default_rng(77)
    for i in range(20):  # cap and threshold (:92-102)
        n = 10 + 3 * i
        eu, ev, ew = rand_edges(rng, n, 0.2, "unit")
        g = B.arrays(n, eu, ev, ew)
        z, trace = B.plp(g, theta=-1, max_iterations=100)
        assert len(trace) <= 100 and trace[-1] <= max(1, n // 100000)
    eu, ev, ew = rand_edges(np.random.default_rng(13), 40, 0.15, "unit")
    g = B.arrays(40, eu, ev, ew)  # determinism (:104-115)
    assert np.array_equal(B.plp(g, theta=0, seed=7)[0], B.plp(g, theta=0, seed=7)[0])


# ---------------------------------------------------------------------------
# T/test_louvain.cpp
# ---------------------------------------------------------------------------
def kat_coarsen(B):
    bar = B.graph(6, BARBELL)
    cg, pi = B.coarsen(bar, TRIANGLES)  # (:101-111)
    c = B.csr(cg)
    assert c["n"] == 2 and c["total"] == 7.0
    assert c["loop"][0] == 3.0 and c["loop"][1] == 3.0 and c["vol"][0] == 7.0 and c["vol"][1] == 7.0
    assert np.array_equal(pi, TRIANGLES)
    ident, _ = B.coarsen(bar, np.arange(6, dtype=np.int32))  # identity (:113-121)
    ci, cb = B.csr(ident), B.csr(bar)
    assert np.array_equal(ci["off"], cb["off"]) and np.array_equal(ci["col"], cb["col"])
    assert np.array_equal(ci["w"], cb["w"])
    one, _ = B.coarsen(bar, np.zeros(6, np.int32))
    assert B.csr(one)["n"] == 1 and B.csr(one)["loop"][0] == 7.0
    with pytest.raises(B.InvalidArgument):  # non-compact (:123-129)
        B.coarsen(bar, np.array([5, 5, 5, 9, 9, 9], np.int32))


def kat_coarsen_invariants(B):
    rng = np.random.default_rng(888)
    for i in range(50):  # (:131-145)
        n = 4 + i % 16
        eu, ev, ew = rand_edges(rng, n, 0.4, "int", loop_p=0.2)
        g = B.arrays(n, eu, ev, ew)
        z = B.compact(rng.integers(0, 1 + i % 5, n).astype(np.int32))[0]
        cg, _ = B.coarsen(g, z)
        c, f = B.csr(cg), B.csr(g)
        assert c["total"] == pytest.approx(f["total"], rel=1e-9)
        assert np.sum(c["vol"]) == pytest.approx(np.sum(f["vol"]), rel=1e-9)
        assert B.modularity(cg, np.arange(c["n"], dtype=np.int32)) == pytest.approx(B.modularity(g, z), abs=1e-9)


def kat_prolong(B):
    assert list(B.prolong([4, 9], [0, 0, 0, 1, 1, 1])) == [4, 4, 4, 9, 9, 9]  # (:158-171)
    assert list(B.prolong([4, 9], [0, 1])) == [4, 9]
    with pytest.raises(B.OutOfRange):
        B.prolong([4, 9], [0, 2])


def kat_plm(B):
    z, q = B.plm(B.graph(6, TWO_TRIANGLES))  # (:183-190)
    assert q == pytest.approx(0.5, abs=1e-12)
    z, q = B.plm(B.graph(6, BARBELL))
    assert q == pytest.approx(5.0 / 14.0, abs=1e-12) and same_relation(z, TRIANGLES)
    z, q = B.plm(B.graph(2, [(0, 1, 1)]))  # single edge (:192-197)
    assert len(set(z.tolist())) == 1 and q == pytest.approx(0.0, abs=1e-15)
    with pytest.raises(B.DomainError):  # edgeless (:199-202)
        B.plm(B.graph(3, []))
    z, q = B.plm(B.graph(6, TWO_TRIANGLES), refine=True)  # PLMR (:235-239)
    assert q == pytest.approx(0.5, abs=1e-12)


def kat_plm_gamma_endpoints(B):
    rng = np.random.default_rng(246)
    for i in range(10):  # (:204-221)
        n = 8 + i
        eu, ev, ew = rand_edges(rng, n, 0.3, "int")
        g = B.arrays(n, eu, ev, ew)
        z0, _ = B.plm(g, gamma=0.0)
        for u, v in zip(eu, ev):
            assert z0[u] == z0[v]
        g1 = B.arrays(n, eu, ev, np.ones(len(eu)))
        zs, _ = B.plm(g1, gamma=2.0 * B.csr(g1)["total"])
        assert len(set(zs.tolist())) == n


def kat_plmr_vs_plm(B):
    rng = np.random.default_rng(135)
    for i in range(25):  # (:223-233)
        n = 10 + i % 15
        eu, ev, ew = rand_edges(rng, n, 0.3, "int", loop_p=0.1)
        g = B.arrays(n, eu, ev, ew)
        _, qp = B.plm(g, seed=i)
        _, qr = B.plm(g, refine=True, seed=i)
        assert qr >= qp - 1e-12


# ---------------------------------------------------------------------------
# T/test_ensemble.cpp, T/test_generator.cpp
# ---------------------------------------------------------------------------
def kat_combine(B):
    a = np.array([0, 0, 1, 1], np.int32)
    b = np.array([0, 1, 1, 0], np.int32)
    out, k = B.combine([a, b])  # (:18-32)
    assert k == 4
    out, k = B.combine([a])
    assert same_relation(out, a)
    rng = np.random.default_rng(4096)
    for i in range(200):  # hashed == exact meet (:70-84)
        n = 4 + i % 20
        sols = [rng.integers(0, 3, n).astype(np.int32) for _ in range(2 + i % 3)]
        out, _ = B.combine(sols)
        tup = np.stack(sols, 1)
        _, exact = np.unique(tup, axis=0, return_inverse=True)
        assert same_relation(out, exact.ravel())
    out, _ = B.combine([np.array([3, 7, 3, 7], np.int32), np.array([1, 2, 1, 2], np.int32)])  # (:86-96)
    assert out[0] == out[2] and out[1] == out[3] and out[0] != out[1]
    with pytest.raises(B.InvalidArgument):  # (:34-39)
        B.combine([np.zeros(3, np.int32), np.zeros(4, np.int32)])


def kat_epp(B):
    z, q = B.epp(B.graph(6, TWO_TRIANGLES))  # (:112-119)
    assert q == pytest.approx(0.5, abs=1e-12)
    with pytest.raises(B.DomainError):  # (:143-150)
        B.epp(B.graph(3, []))
    with pytest.raises(B.InvalidArgument):
        B.epp(B.graph(6, BARBELL), b=0)


def kat_epp_refines_core(B):
    rng = np.random.default_rng(21)
    for i in range(10):  # output refines... core refines output (:121-141)
        n = 20 + 3 * i
        eu, ev, ew = rand_edges(rng, n, 0.2, "unit")
        g = B.arrays(n, eu, ev, ew)
        seed = 100 + i
        bases = [B.plp(g, seed=seed + b)[0] for b in range(3)]
        core, _ = B.combine(bases)
        z, _ = B.epp(g, b=3, seed=seed)
        assert refines(core, z)


def kat_generator(B):
    g, truth = B.planted(6, 2, 1.0, 0.0, 1)  # (:12-17)
    c, t = B.csr(g), B.csr(B.graph(6, TWO_TRIANGLES))
    assert np.array_equal(c["off"], t["off"]) and np.array_equal(c["col"], t["col"])
    assert same_relation(truth, TRIANGLES)
    g, truth = B.planted(10, 2, 0.0, 0.0, 1)  # (:19-24)
    assert B.csr(g)["m"] == 0 and B.csr(g)["n"] == 10
    for spec in [(10, 0, 0.5, 0.1, 1), (10, 11, 0.5, 0.1, 1), (10, 2, 0.1, 0.5, 1), (10, 2, 1.5, 0.1, 1)]:
        with pytest.raises(B.InvalidArgument):  # (:26-31)
            B.planted(*spec)
    g1, t1 = B.planted(300, 5, 0.2, 0.01, 7)  # determinism (:33-41)
    g2, t2 = B.planted(300, 5, 0.2, 0.01, 7)
    assert np.array_equal(B.csr(g1)["col"], B.csr(g2)["col"]) and np.array_equal(t1, t2)
    g, truth = B.planted(103, 10, 0.0, 0.0, 1)  # blocks near-equal (:43-52)
    sizes = np.bincount(truth)
    assert len(sizes) == 10 and sizes.min() >= 10 and sizes.max() <= 11
    g, truth = B.planted(200, 4, 0.3, 0.05, 11)  # invariants (:75-82)
    c = B.csr(g)
    assert np.sum(c["vol"]) == pytest.approx(2.0 * c["total"], rel=1e-12)


ALL = [kat_graph_counts, kat_graph_errors, kat_graph_random_invariants, kat_modularity_known,
       kat_modularity_identity, kat_dominant_label, kat_plp_runs, kat_plp_random, kat_coarsen,
       kat_coarsen_invariants, kat_prolong, kat_plm, kat_plm_gamma_endpoints, kat_plmr_vs_plm, kat_combine, kat_epp,
       kat_epp_refines_core, kat_generator]
