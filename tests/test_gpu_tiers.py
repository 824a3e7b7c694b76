"""Every degree tier of the sweep / move kernels on one graph, bit-exact
against the oracle: a sparse random base plus hub nodes whose degrees land in
BLOCK2 (<= 4096), BLOCK3 (<= 8192), CLUSTER (<= 32768, integer tallies) and
HUB (larger), for count, integer and dyadic-real weights (the three tally
classes).  Checked: synchronous PLP sweeps, the move evaluation (best label
and gain), and PLP / PLM / PLMR end to end."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HUB_DEGREES = (3000, 6000, 9000, 20000, 31000, 40000)


def _tier_graph(oracle, kind, seed=4, n=60000):
    rng = np.random.default_rng(seed)
    m0 = 3 * n
    eu = rng.integers(0, n, m0)
    ev = rng.integers(0, n, m0)
    keep = eu != ev
    eu, ev = eu[keep], ev[keep]
    hubs = rng.choice(n, size=len(HUB_DEGREES), replace=False)
    for h, d in zip(hubs, HUB_DEGREES):
        nb = rng.choice(n, size=d + 1, replace=False)
        nb = nb[nb != h][:d]
        eu = np.concatenate([eu, np.full(len(nb), h)])
        ev = np.concatenate([ev, nb])
    a, b = np.minimum(eu, ev), np.maximum(eu, ev)
    key = np.unique(a.astype(np.int64) * n + b)
    eu, ev = (key // n).astype(np.int32), (key % n).astype(np.int32)
    if kind == "count":
        ew = np.ones(len(eu))
    elif kind == "int":
        ew = rng.integers(1, 6, len(eu)).astype(np.float64)
    else:
        ew = (rng.integers(0, 1 << 24, len(eu)) + 1) * 2.0 ** -24
    og = oracle.from_arrays(n, eu, ev, ew)
    return og, hubs


def _dev_graph(dev, og, kind):
    w = None if kind == "count" else og.w.astype(np.float32)
    return dev.Graph.from_csr(og.n, og.off, og.col, w)


@pytest.fixture(scope="module", params=["count", "int", "real"])
def tier_case(request, oracle):
    og, hubs = _tier_graph(oracle, request.param)
    return request.param, og, hubs


def test_degrees_cover_all_tiers(tier_case):
    _, og, hubs = tier_case
    deg = np.diff(og.off)
    for h, d in zip(hubs, HUB_DEGREES):
        assert deg[h] >= d
    assert deg.max() > 32768 and ((deg > 4096) & (deg <= 8192)).any() and ((deg > 8192) & (deg <= 32768)).any()


def test_sync_sweeps_all_tiers(dev, ctx, oracle, tier_case):
    kind, og, _ = tier_case
    g = _dev_graph(dev, og, kind)
    z = np.arange(og.n, dtype=np.int32)
    for it in range(3):
        ref_out, ref_upd = oracle.plp_sweep_sync(og, z)
        out, upd = dev.plp_sweep_sync(g, z)
        assert upd == ref_upd and np.array_equal(out, ref_out), f"sweep {it}"
        z = ref_out


def test_move_eval_all_tiers(dev, ctx, oracle, tier_case):
    kind, og, _ = tier_case
    g = _dev_graph(dev, og, kind)
    z, _ = oracle.move_phase_bucketed(og, np.arange(og.n, dtype=np.int32), salt=0, max_move_iterations=2)
    zc, _ = oracle.compact(z)
    vols = oracle.community_volumes(og, zc, ub=og.n)
    best_ref, gain_ref = oracle.move_eval(og, zc, vols)
    best, gain = dev.move_eval(g, zc, vols)
    assert np.array_equal(best, best_ref)
    np.testing.assert_array_equal(gain, gain_ref)


def test_end_to_end_all_tiers(dev, ctx, oracle, tier_case):
    kind, og, _ = tier_case
    g = _dev_graph(dev, og, kind)
    lab_ref, trace_ref = oracle.plp_bucketed(og, seed=6)
    lab, rep = dev.run_plp(g, dev.PlpConfig(seed=6))
    assert [it["updated"] for it in rep.iterations] == trace_ref.tolist()
    assert np.array_equal(lab, lab_ref)
    for refine in (False, True):
        z_ref, k_ref, _ = oracle.louvain_bucketed(og, refine=refine, seed=8)
        z, rep = dev.run_louvain(g, dev.LouvainConfig(refine=refine, seed=8))
        assert np.array_equal(z, z_ref), f"refine={refine}"
        assert rep.community_count == k_ref
