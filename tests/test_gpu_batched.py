"""Bounded-scratch paths for graphs near the device's capacity (C5: R-MAT
scale 28, 8.5e9 entries on one B200): the contraction split into batches of
coarse rows (CD_COARSEN_CHUNK_ENTRIES) must give exactly the one-batch coarse
graph -- and therefore the same detector output -- and is pinned against the
oracle's coarsen on the same partition."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("weighted", [False, True])
def test_batched_contraction_equals_single(dev, ctx, oracle, monkeypatch, weighted):
    g = dev.generate_rmat(13, 8, weighted=weighted, seed=2, ctx=ctx)
    z, _ = dev.run_plm(g, dev.LouvainConfig(seed=1))
    z = np.array(z)
    cg1, pi1 = dev.coarsen(g, z)
    ref = cg1.csr()
    for chunk, keep in (("50000", None), ("3000", None), ("3000", "0"), ("20000", "100000"), ("1", None)):
        monkeypatch.setenv("CD_COARSEN_CHUNK_ENTRIES", chunk)
        if keep is None:
            monkeypatch.delenv("CD_COARSEN_KEEP_BYTES", raising=False)
        else:  # batches beyond the budget are recomputed in pass B
            monkeypatch.setenv("CD_COARSEN_KEEP_BYTES", keep)
        cg, pi = dev.coarsen(g, z)
        c = cg.csr()
        assert np.array_equal(pi, pi1)
        for key in ref:
            np.testing.assert_array_equal(c[key], ref[key], err_msg=f"{key} chunk={chunk}")
        assert cg.edge_count() == cg1.edge_count() and cg.total_edge_weight() == cg1.total_edge_weight()
    # pinned: the oracle's contraction of the same partition
    c = g.csr()
    og = oracle.from_csr(g.node_count(), c["off"], c["col"], c["w"])
    ocg = oracle.coarsen(og, z)
    assert np.array_equal(ref["off"], ocg.off) and np.array_equal(ref["col"], ocg.col)
    np.testing.assert_allclose(ref["w"], ocg.w, rtol=1e-6)


def test_batched_contraction_in_detectors(dev, ctx, monkeypatch):
    g = dev.generate_rmat(13, 8, seed=5, ctx=ctx)
    z1, r1 = dev.run_plm(g, dev.LouvainConfig(seed=3))
    monkeypatch.setenv("CD_COARSEN_CHUNK_ENTRIES", "20000")
    monkeypatch.setenv("CD_BUILD_CHUNK_ENTRIES", "30000")
    monkeypatch.setenv("CD_COARSEN_KEEP_BYTES", "200000")
    g2 = dev.generate_rmat(13, 8, seed=5, ctx=ctx)
    z2, r2 = dev.run_plm(g2, dev.LouvainConfig(seed=3))
    assert np.array_equal(np.array(z1), np.array(z2)) and r1.modularity == r2.modularity
