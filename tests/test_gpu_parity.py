"""Parity of the CUDA path (through the C ABI) with the oracle.

Deterministic sub-kernels must match exactly (north_star): one synchronous
PLP sweep (labels bit-exact), contraction by a given partition (integer
structure bit-exact, fp32 weights within 1e-6 relative of the fp64
reference), modularity of a given partition (within 1e-6 relative; we test
1e-9).  The move evaluation, compaction, combine and generators are
bit-exact too.  End-to-end drivers are bit-exact against the C port of the
same bucketed order (oracle/commdet_oracle.c) and within 0.005 modularity of
the reference itself (oracle/_ref).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL_W = 1e-6    # north_star: float weights within 1e-6 relative
REL_Q = 1e-6    # north_star: modularity within 1e-6 relative
E2E_Q = 0.005   # north_star: end-to-end modularity within 0.005 absolute


def dev_graph_from_csr(dev, g):
    w = None if np.all(g.w == 1.0) else g.w.astype(np.float32)
    return dev.Graph.from_csr(g.n, g.off, g.col, w)


def assert_csr_equal(dev_g, og, weights_exact=True):
    c = dev_g.csr()
    assert np.array_equal(c["off"], og.off)
    assert np.array_equal(c["col"], og.col)
    w = c["w"].astype(np.float64) if c["w"] is not None else np.ones(len(c["col"]))
    if weights_exact:
        np.testing.assert_array_equal(w, og.w)
    else:
        np.testing.assert_allclose(w, og.w, rtol=REL_W)
    rel = 1e-12 if weights_exact else REL_W
    np.testing.assert_allclose(c["vol"], og.vol, rtol=rel)
    np.testing.assert_allclose(c["loop"], og.loop, rtol=rel)
    assert dev_g.edge_count() == og.m
    assert dev_g.total_edge_weight() == pytest.approx(og.total, rel=rel)


# ---------------------------------------------------------------------------
# golden vectors (reference-generated)
# ---------------------------------------------------------------------------
def test_golden_builder_sweep_modularity_coarsen(golden, dev, ctx, oracle):
    arr, man = golden
    for c in man["cases"]:
        k = c["key"]
        n = len(arr[f"{k}_vol"])
        g = dev.Graph.from_edges(n, (arr[f"{k}_eu"], arr[f"{k}_ev"], arr[f"{k}_ew"].astype(np.float32)))
        og = oracle.from_arrays(n, arr[f"{k}_eu"], arr[f"{k}_ev"], arr[f"{k}_ew"])
        assert_csr_equal(g, og)
        z = arr[f"{k}_z"]
        for gamma, q in c["modularity"].items():
            assert dev.modularity(g, z, float(gamma), ub=c["k"]) == pytest.approx(q, rel=1e-9, abs=1e-12)
        assert dev.coverage(g, z) == pytest.approx(c["coverage"], abs=1e-12)
        for tag, lab in (("s", np.arange(n, dtype=np.int32)), ("z", z)):
            out, upd = dev.plp_sweep_sync(g, lab)
            assert np.array_equal(out, arr[f"{k}_sweep_{tag}"]), (k, tag)
            assert upd == int(np.sum(out != lab))
        zc, kk = dev.compacted(z)
        assert np.array_equal(zc, arr[f"{k}_zc"])
        cg, pi = dev.coarsen(g, arr[f"{k}_zc"])
        cc = cg.csr()
        assert np.array_equal(cc["off"], arr[f"{k}_coff"]) and np.array_equal(cc["col"], arr[f"{k}_ccol"])
        np.testing.assert_allclose(cc["w"], arr[f"{k}_cw"], rtol=REL_W)
        # coarse weights are stored as fp32 (one rounding), so vol follows them
        np.testing.assert_allclose(cc["vol"], arr[f"{k}_cvol"], rtol=REL_W)
        assert cg.edge_count() == c["cm"] and cg.total_edge_weight() == pytest.approx(c["ctotal"], rel=REL_W)
        assert np.array_equal(pi, arr[f"{k}_zc"])


def test_golden_planted_and_combine(golden, dev, ctx):
    arr, man = golden
    for p in man["planted"]:
        g, truth = dev.generate_planted(*p["spec"])
        c = g.csr()
        assert g.edge_count() == p["m"]
        assert np.array_equal(c["off"], arr[f"{p['key']}_off"]) and np.array_equal(c["col"], arr[f"{p['key']}_col"])
        assert np.array_equal(truth, arr[f"{p['key']}_truth"])
    out, k = dev.combine_hashed([arr[f"ens_sol{j}"] for j in range(4)])
    assert np.array_equal(out, arr["ens_hashed"])


# ---------------------------------------------------------------------------
# generators vs the C port (identical bytes)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("weighted", [False, True])
def test_rmat_generator_bit_exact(dev, ctx, oracle, weighted):
    og = oracle.generate_rmat(14, 16, weighted=weighted, seed=3)
    g = dev.generate_rmat(14, 16, weighted=weighted, seed=3)
    assert_csr_equal(g, og)


def test_lfr_generator_bit_exact(dev, ctx, oracle):
    og, ot = oracle.generate_lfr(seed=5, n=20000)
    g, t = dev.generate_lfr(seed=5, n=20000)
    assert np.array_equal(t, ot)
    assert_csr_equal(g, og)


def test_planted_c1_generator_matches_reference(dev, ctx, ref):
    """Config 1 edge set is bit-identical to generate_planted (m = 594,718)."""
    rg, rt = ref.RefGraph.planted(100000, 1000, 0.1, 2 / 99900, 1, workers=0)
    c = rg.csr()
    g, truth = dev.generate_planted(100000, 1000, 0.1, 2 / 99900, 1)
    d = g.csr()
    assert g.edge_count() == c.m == 594718
    assert np.array_equal(d["off"], c.off) and np.array_equal(d["col"], c.col)
    assert np.array_equal(truth, rt)


# ---------------------------------------------------------------------------
# deterministic sub-kernels at scale (all degree tiers incl. hubs)
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def rmat18(oracle):
    return {w: oracle.generate_rmat(18, 16, weighted=w, seed=11) for w in (False, True)}


@pytest.mark.parametrize("weighted", [False, True])
def test_sync_sweep_rmat_all_tiers(dev, ctx, oracle, rmat18, weighted):
    og = rmat18[weighted]
    g = dev.generate_rmat(18, 16, weighted=weighted, seed=11)
    assert g.max_degree > 4096  # hub tier exercised
    z = np.arange(og.n, dtype=np.int32)
    for it in range(4):
        ref_out, ref_upd = oracle.plp_sweep_sync(og, z)
        out, upd = dev.plp_sweep_sync(g, z)
        assert upd == ref_upd
        assert np.array_equal(out, ref_out), f"sweep {it}"
        z = ref_out


@pytest.mark.parametrize("weighted", [False, True])
def test_modularity_move_eval_coarsen_rmat(dev, ctx, oracle, rmat18, weighted):
    og = rmat18[weighted]
    g = dev.generate_rmat(18, 16, weighted=weighted, seed=11)
    # a Louvain-like partition: one bucketed move phase from singletons
    z, _ = oracle.move_phase_bucketed(og, np.arange(og.n, dtype=np.int32), salt=0, max_move_iterations=3)
    zc, k = oracle.compact(z)
    q_ref = oracle.modularity(og, zc)
    assert dev.modularity(g, zc) == pytest.approx(q_ref, rel=1e-9)
    assert dev.coverage(g, zc) == pytest.approx(oracle.coverage(og, zc), rel=1e-9)
    vols = oracle.community_volumes(og, zc, ub=og.n)
    best_ref, gain_ref = oracle.move_eval(og, zc, vols)
    best, gain = dev.move_eval(g, zc, vols)
    assert np.array_equal(best, best_ref)
    np.testing.assert_array_equal(gain, gain_ref)
    cg, pi = dev.coarsen(g, zc)
    ocg = oracle.coarsen(og, zc)
    assert_csr_equal(cg, ocg, weights_exact=False)
    # the coarse graph carries fp32-rounded weights: Q agrees to ~1e-7
    assert dev.modularity(cg, np.arange(k, dtype=np.int32)) == pytest.approx(q_ref, rel=REL_Q)


def test_modularity_vs_reference_flooded_partition(dev, ctx, ref, rmat18):
    """Catastrophic cancellation case (SURVEY finding 11): PLP floods R-MAT."""
    og = rmat18[False]
    g = dev.generate_rmat(18, 16, weighted=False, seed=11)
    z, _ = dev.run_plp(g)
    rg = ref.RefGraph.from_csr(og)
    zc, _ = dev.compacted(z)
    q_ref, cov_ref = rg.modularity(zc)
    assert dev.modularity(g, zc) == pytest.approx(q_ref, rel=REL_Q)
    assert dev.coverage(g, zc) == pytest.approx(cov_ref, rel=1e-12)


# ---------------------------------------------------------------------------
# end to end: bit-exact vs the C port of the bucketed order
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def e2e_graphs(oracle):
    pg, _ = oracle.generate_planted(2000, 8, 0.05, 0.002, 3)
    lg, _ = oracle.generate_lfr(seed=2, n=20000)
    rg = oracle.generate_rmat(14, 16, weighted=True, seed=9)
    ru = oracle.generate_rmat(17, 16, weighted=False, seed=4)  # hubs; PLP's margin-pruned active set
    return {"planted": pg, "lfr": lg, "rmat_w": rg, "rmat_u": ru}


def _dev_of(dev, name, og):
    if name == "planted":
        return dev.generate_planted(2000, 8, 0.05, 0.002, 3)[0]
    if name == "lfr":
        return dev.generate_lfr(seed=2, n=20000)[0]
    if name == "rmat_u":
        return dev.generate_rmat(17, 16, weighted=False, seed=4)
    return dev.generate_rmat(14, 16, weighted=True, seed=9)


@pytest.mark.parametrize("name", ["planted", "lfr", "rmat_w", "rmat_u"])
def test_plp_end_to_end_bit_exact(dev, ctx, oracle, e2e_graphs, name):
    og = e2e_graphs[name]
    g = _dev_of(dev, name, og)
    lab_ref, trace_ref = oracle.plp_bucketed(og, seed=5)
    lab, rep = dev.run_plp(g, dev.PlpConfig(seed=5))
    assert [it["updated"] for it in rep.iterations] == trace_ref.tolist()
    assert np.array_equal(lab, lab_ref)
    assert rep.modularity == pytest.approx(oracle.modularity(og, oracle.compact(lab_ref)[0]), rel=1e-9)
    assert rep.community_count == oracle.community_count(lab_ref)


@pytest.mark.parametrize("name", ["planted", "lfr", "rmat_w"])
@pytest.mark.parametrize("refine", [False, True])
def test_louvain_end_to_end_bit_exact(dev, ctx, oracle, e2e_graphs, name, refine):
    og = e2e_graphs[name]
    g = _dev_of(dev, name, og)
    z_ref, k_ref, lv_ref = oracle.louvain_bucketed(og, refine=refine, seed=3)
    z, rep = dev.run_louvain(g, dev.LouvainConfig(refine=refine, seed=3))
    assert np.array_equal(z, z_ref)
    assert rep.community_count == k_ref and len(rep.levels) == lv_ref
    assert rep.modularity == pytest.approx(oracle.modularity(og, z_ref), rel=1e-9)


@pytest.mark.parametrize("name", ["planted", "lfr"])
def test_epp_end_to_end_bit_exact(dev, ctx, oracle, e2e_graphs, name):
    og = e2e_graphs[name]
    g = _dev_of(dev, name, og)
    z_ref, k_ref = oracle.epp_bucketed(og, ensemble_size=4, seed=2)
    z, rep = dev.run_epp(g, dev.EnsembleConfig(ensemble_size=4, seed=2))
    assert np.array_equal(z, z_ref)
    assert rep.community_count == k_ref


# ---------------------------------------------------------------------------
# end to end vs the reference itself (quality within 0.005)
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c1(ref):
    rg, truth = ref.RefGraph.planted(100000, 1000, 0.1, 2 / 99900, 1, workers=0)
    return rg, truth


def test_c1_plp_quality_vs_reference(dev, ctx, c1):
    rg, _ = c1
    g, _ = dev.generate_planted(100000, 1000, 0.1, 2 / 99900, 1)
    _, rrep, _ = rg.run_plp(randomize=True, seed=1, workers=1)  # the named parity setting
    lab, rep = dev.run_plp(g)
    assert abs(rep.modularity - rrep["modularity"]) <= E2E_Q
    assert rep.community_count > 0


@pytest.mark.parametrize("refine", [False, True])
def test_c1_louvain_quality_vs_reference(dev, ctx, c1, refine):
    rg, _ = c1
    g, _ = dev.generate_planted(100000, 1000, 0.1, 2 / 99900, 1)
    _, rrep = rg.run_louvain(refine=refine, workers=1)
    z, rep = dev.run_louvain(g, dev.LouvainConfig(refine=refine))
    assert abs(rep.modularity - rrep["modularity"]) <= E2E_Q


def test_c1_epp_quality_vs_reference(dev, ctx, c1):
    rg, _ = c1
    g, _ = dev.generate_planted(100000, 1000, 0.1, 2 / 99900, 1)
    # one worker: the reference's multi-threaded EPP varies from run to run
    # (racing PLP bases), which made this comparison flaky
    _, rrep = rg.run_epp(workers=1)
    z, rep = dev.run_epp(g)
    assert abs(rep.modularity - rrep["modularity"]) <= E2E_Q


@pytest.mark.parametrize("name", ["planted", "lfr", "rmat_w"])
def test_louvain_reference_stopping_bit_exact(dev, ctx, oracle, e2e_graphs, name):
    """cd_louvain_config_reference: the reference's stopping rule alone
    (H/louvain.hpp:78, :136-137), no pruning -- bit-exact vs the port."""
    og = e2e_graphs[name]
    g = _dev_of(dev, name, og)
    kw = dict(move_theta=0, move_tol=0.0, move_stall=0.0, prune=False, move_qtol=0.0)
    z_ref, k_ref, lv_ref = oracle.louvain_bucketed(og, seed=3, **kw)
    z, rep = dev.run_louvain(g, dev.LouvainConfig.reference(seed=3))
    assert np.array_equal(z, z_ref)
    assert rep.community_count == k_ref and len(rep.levels) == lv_ref


@pytest.mark.parametrize("kind", ["unit", "int", "dyadic"])
def test_end_to_end_with_loops_and_isolated_nodes(dev, ctx, oracle, kind):
    """Self-loops, isolated nodes and every weight kind through the first
    sub-sweeps from singletons (PLP's row-first-entry rule, PLM's tally-free
    evaluation) and the margin-pruned active set: bit-exact vs the port."""
    from conftest import rand_edges
    rng = np.random.default_rng(17)
    n = 3000
    eu, ev, ew = rand_edges(rng, n, 0.004, kind=kind, loop_p=0.2)
    keep = (eu < n - 100) & (ev < n - 100)  # the last 100 nodes stay isolated
    eu, ev, ew = eu[keep], ev[keep], ew[keep]
    og = oracle.from_arrays(n, eu, ev, ew)
    w = None if kind == "unit" else ew.astype(np.float32)
    g = dev.Graph.from_edges(n, (eu, ev, w)) if w is not None else dev.Graph.from_edges(n, (eu, ev))
    lab_ref, trace_ref = oracle.plp_bucketed(og, seed=4)
    lab, rep = dev.run_plp(g, dev.PlpConfig(seed=4))
    assert [it["updated"] for it in rep.iterations] == trace_ref.tolist()
    assert np.array_equal(lab, lab_ref)
    for refine in (False, True):
        z_ref, k_ref, _ = oracle.louvain_bucketed(og, refine=refine, seed=4)
        z, rep = dev.run_louvain(g, dev.LouvainConfig(refine=refine, seed=4))
        assert np.array_equal(z, z_ref), refine


def test_uint64_iteration_caps_saturate(dev, ctx, oracle, e2e_graphs):
    """The reference's caps are uint64 counts (H/plp.hpp:20, H/louvain.hpp:17):
    UINT64_MAX means "until converged" -- it saturates, never wraps to -1
    (zero iterations) or truncates, and the per-pass trace stays bounded."""
    og = e2e_graphs["lfr"]
    g = _dev_of(dev, "lfr", og)
    big = (1 << 64) - 1
    lab, rep = dev.run_plp(g, dev.PlpConfig(seed=5, max_iterations=big))
    lab_ref, trace_ref = oracle.plp_bucketed(og, seed=5)
    assert np.array_equal(lab, lab_ref) and len(rep.iterations) == len(trace_ref)
    z, rep = dev.run_louvain(g, dev.LouvainConfig(seed=3, max_move_iterations=big, max_levels=big))
    z_ref, _, _ = oracle.louvain_bucketed(og, seed=3)
    assert np.array_equal(z, z_ref)
    # 2^32 + 1 passes is not 1 pass
    z2, _ = dev.run_louvain(g, dev.LouvainConfig(seed=3, max_move_iterations=(1 << 32) + 1))
    assert np.array_equal(z2, z_ref)
