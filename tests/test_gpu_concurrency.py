"""Concurrent EPP bases (csrc/detect.cu): on one device the PLP bases run
at the same time, one host thread and child context each (own stream,
counters and hub-tier scratch; the graph's work decomposition shared
read-only).  The result must equal the serial run's bit for bit, including
graphs whose hubs use the partitioned HUB tier (real weights, degree > 8192)
-- the scratch the concurrent runs must not share."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("weighted,scale", [(True, 16), (False, 14)])
def test_concurrent_bases_equal_serial(dev, ctx, monkeypatch, weighted, scale):
    g = dev.generate_rmat(scale, 16, weighted=weighted, seed=3, ctx=ctx)
    assert g.max_degree > 256  # the concurrent path's condition
    if weighted:
        assert g.max_degree > 8192  # HUB tier for fp64 tallies
    cfg = dev.EnsembleConfig(ensemble_size=4, seed=5)
    monkeypatch.setenv("CD_EPP_CONCURRENT", "0")
    z0, r0 = dev.run_epp(g, cfg)
    monkeypatch.setenv("CD_EPP_CONCURRENT", "1")
    for _ in range(2):
        z1, r1 = dev.run_epp(g, cfg)
        assert np.array_equal(np.array(z1), np.array(z0))
        assert r1.community_count == r0.community_count
        assert r1.modularity == pytest.approx(r0.modularity, rel=1e-12, abs=1e-15)
    # kernel launches of the child contexts are accounted to the caller's
    assert r1.kernel_launches > 0
