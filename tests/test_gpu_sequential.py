"""MoveObserver and EnsembleConfig::base_override on the device.

* cd_move_phase_sequential (the reference's one-worker move phase,
  H/louvain.hpp:65-141) against the oracle's restatement, which
  tests/test_oracle_sequential.py pins to the reference itself: final labels
  and the whole observed move sequence (node, source, target, gain) bit-exact
  for unit, integer and real weights.
* the observer sees every move applied (T/test_louvain.cpp:85-98,
  acceptance criterion 6): modularity strictly rises move by move.
* cd_epp_run_bases (H/ensemble.hpp:127-128): singleton bases give plain PLM
  (T/test_ensemble.cpp:101-113); bases equal to the device's own PLP runs
  give run_epp's labels exactly."""
import numpy as np
import pytest

from conftest import rand_edges

pytestmark = pytest.mark.gpu


def _pair(dev, oracle, seed, n, p, kind, loop_p=0.1):
    rng = np.random.default_rng(seed)
    eu, ev, ew = rand_edges(rng, n, p, kind, loop_p)
    og = oracle.from_arrays(n, eu, ev, ew)
    w = None if kind == "unit" else og.w.astype(np.float32)
    return dev.Graph.from_csr(og.n, og.off, og.col, w), og


@pytest.mark.parametrize("kind", ["unit", "int", "real"])
def test_sequential_move_phase_bit_exact(dev, ctx, oracle, kind):
    for i in range(8):
        g, og = _pair(dev, oracle, 500 + i, 8 + 9 * i, 0.3 if i < 4 else 0.06, kind)
        z0 = np.arange(og.n, dtype=np.int32)
        seen = []
        z, ch = dev.move_phase_sequential(g, z0.copy(), observer=lambda u, c, d, gain: seen.append((u, c, d, gain)))
        zo, cho, moves = oracle.move_phase_sequential(og, z0)
        assert ch == cho
        assert np.array_equal(z, zo), f"case {i}"
        assert seen == moves, f"case {i}"


def test_sequential_move_phase_larger_graphs(dev, ctx, oracle):
    # an LFR-shaped graph (hubs over 32 entries: multi-chunk rows) and a planted one,
    # from a non-singleton start with a pass cap
    og, _ = oracle.generate_lfr(seed=3, n=3000, avg_degree=12, max_degree=150, min_community=20, max_community=200)
    g = dev.Graph.from_csr(og.n, og.off, og.col)
    rng = np.random.default_rng(5)
    z0 = rng.integers(0, 400, og.n).astype(np.int32)
    for cap in (1, 3, 32):
        z, ch = dev.move_phase_sequential(g, z0.copy(), dev.LouvainConfig(max_move_iterations=cap), ub=400)
        zo, cho, _ = oracle.move_phase_sequential(og, z0, max_move_iterations=cap, ub=400)
        assert ch == cho and np.array_equal(z, zo), cap
    pg, _ = oracle.generate_planted(2000, 20, 0.05, 0.002, 9)
    g2 = dev.Graph.from_csr(pg.n, pg.off, pg.col)
    z0 = np.arange(pg.n, dtype=np.int32)
    z, _ = dev.move_phase_sequential(g2, z0.copy(), dev.LouvainConfig(gamma=0.7))
    zo, _, _ = oracle.move_phase_sequential(pg, z0, gamma=0.7)
    assert np.array_equal(z, zo)


def test_observer_sees_monotone_modularity(dev, ctx, oracle):
    rng = np.random.default_rng(404)
    total = 0
    for i in range(20):
        n = 8 + i % 12
        eu, ev, ew = rand_edges(rng, n, 0.35, "unit")
        g = dev.Graph.from_edges(n, list(zip(eu.tolist(), ev.tolist(), ew.tolist())))
        z = np.arange(n, dtype=np.int32)
        last = [dev.modularity(g, z)]

        def obs(u, c, d, gain):
            assert z[u] == d and c != d and gain > 0
            now = dev.modularity(g, z, ub=n)
            assert now > last[0]
            last[0] = now

        out, _ = dev.move_phase_sequential(g, z, observer=obs)
        assert out is z  # updated in place, like the reference's Partition&
        total += 1
    assert total == 20


def test_sequential_errors(dev, ctx, oracle):
    g, og = _pair(dev, oracle, 1, 12, 0.3, "unit")
    with pytest.raises(dev.OutOfRange):
        dev.move_phase_sequential(g, np.full(og.n, 20, np.int32), ub=12)
    with pytest.raises(dev.InvalidArgument):
        dev.move_phase_sequential(g, np.zeros(og.n + 1, np.int32))

    def boom(*_):
        raise KeyError("observer")

    with pytest.raises(KeyError):
        dev.move_phase_sequential(g, np.arange(og.n, dtype=np.int32), observer=boom)
    # no edges: nothing moves
    e = dev.Graph.from_edges(4, [])
    z, ch = dev.move_phase_sequential(e, np.arange(4, dtype=np.int32))
    assert not ch and np.array_equal(z, np.arange(4))


def test_epp_singleton_base_override_equals_plm(dev, ctx):
    g = dev.Graph.from_edges(6, [(0, 1, 1), (0, 2, 1), (1, 2, 1), (3, 4, 1), (3, 5, 1), (4, 5, 1), (2, 3, 1)])
    calls = []

    def singletons(graph, seed):
        calls.append(seed)
        return np.arange(graph.node_count(), dtype=np.int32)

    cfg = dev.EnsembleConfig(ensemble_size=1, final_algo=dev.ALGO_PLM, workers=1, base_override=singletons)
    z, rep = dev.run_epp(g, cfg)
    zp, rp = dev.run_plm(g, dev.LouvainConfig(workers=1))
    assert calls == [1]
    assert np.array_equal(z, zp)
    assert rep.modularity == pytest.approx(rp.modularity, abs=1e-12)
    assert rep.algorithm == "epp"


def test_epp_base_override_with_device_plp_bases_equals_run_epp(dev, ctx):
    g = dev.generate_rmat(14, 8, seed=3)
    cfg = dev.EnsembleConfig(ensemble_size=4, seed=7)
    z_ref, r_ref = dev.run_epp(g, cfg)

    def plp_base(graph, seed):
        pc = dev.PlpConfig(randomize_order=True, seed=seed)
        return dev.run_plp(graph, pc)[0].copy()

    z, r = dev.run_epp(g, dev.EnsembleConfig(ensemble_size=4, seed=7, base_override=plp_base))
    assert np.array_equal(z, z_ref)
    assert r.modularity == r_ref.modularity and r.community_count == r_ref.community_count
    # the hook's partitions must cover the graph
    bad = dev.EnsembleConfig(ensemble_size=2, base_override=lambda gr, s: np.zeros(gr.node_count() - 1, np.int32))
    with pytest.raises(dev.InvalidArgument):
        dev.run_epp(g, bad)
