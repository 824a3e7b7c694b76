"""Per-kernel work counters behind bench.py's roofline: every sweep / move
kernel family that launched reports algorithmic bytes from its device-side
node and entry tallies (DESIGN.md byte model), the base family carries their
sum, and the hub tier's several kernels are timed as one family."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SLOTS = ("g8", "g16", "g32", "warp", "block", "block2", "block3", "cluster", "hub", "small", "fused")


def _profiled(ctx, fn):
    ctx.reset_stats()
    ctx.set_profiling(True)
    try:
        fn()
    finally:
        ctx.set_profiling(False)
    return ctx.kernel_stats()


def _check_families(stats, base):
    launched = [s for s in SLOTS if f"{base}.{s}" in stats]
    assert launched, f"no {base} kernels profiled"
    total = 0.0
    for s in launched:
        st = stats[f"{base}.{s}"]
        assert st["launches"] > 0 and st["total_ms"] > 0
        assert st["bytes"] > 0, f"{base}.{s} launched with no work counted"
        total += st["bytes"]
    assert stats[base]["bytes"] == pytest.approx(total, rel=1e-12)
    return launched


def test_small_and_tiered_move_counters(dev, ctx, oracle):
    from test_gpu_tiers import _tier_graph, _dev_graph
    og, _ = _tier_graph(oracle, "count")
    g = _dev_graph(dev, og, "count")
    stats = _profiled(ctx, lambda: dev.run_louvain(g, dev.LouvainConfig(seed=3)))
    launched = _check_families(stats, "plm_move")
    # level 0 spans the degree tiers up to the hub; coarse levels fit the
    # one-kernel small move phase
    assert {"hub", "cluster", "small"} <= set(launched)
    hub_parts = [k for k in stats if k.startswith("plm_move.hub_")]
    assert hub_parts
    assert stats["plm_move.hub"]["total_ms"] == pytest.approx(sum(stats[k]["total_ms"] for k in hub_parts))


def test_fused_plp_counters(dev, ctx):
    g, _ = dev.generate_planted(20000, 200, 0.02, 0.0005, seed=5)
    stats = _profiled(ctx, lambda: dev.run_plp(g, dev.PlpConfig(seed=1)))
    launched = _check_families(stats, "plp_sweep")
    assert "fused" in launched
    # a fused PLP run touches every node at least once: >= 17 B per node
    assert stats["plp_sweep.fused"]["bytes"] >= 17 * 20000
