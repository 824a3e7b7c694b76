"""Sharded execution on one GPU through the C ABI.

G ranks are emulated by the loopback transport: G host threads, each with its
own cd_ctx on cuda:0, exchanging through host barriers and stream-ordered
device copies (no kernel waits on another rank; B200_PROFILING.md).  The
sharded drivers evaluate only each rank's nodes and apply every rank's move
list after each sub-sweep, so for unweighted / integer-weight graphs the
labels must be bit-identical to the one-device run -- PLP, PLM, PLMR, EPP,
with replicated graphs and with row shards, coarse levels included
(CD_SHARD_MIN_ENTRIES=0 keeps even tiny coarse graphs on the exchange path).
The NCCL transport itself is exercised at world size 1 (every sub-sweep still
goes through ncclAllGather).
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

JOIN_S = 300


@pytest.fixture(autouse=True)
def _exchange_everywhere(monkeypatch):
    monkeypatch.setenv("CD_SHARD_MIN_ENTRIES", "0")
    monkeypatch.setenv("CD_POOL_RESERVE_FRAC", "0")  # many short-lived contexts


def run_ranks(dev, G, fn):
    """fn(ctx, rank) on G loopback ranks; returns the per-rank results."""
    group = dev.LoopbackGroup(G)
    out, errs = [None] * G, [None] * G

    def work(r):
        ctx = None
        try:
            ctx = dev.Context(0)
            ctx.attach_loopback(group, r)
            out[r] = fn(ctx, r)
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            errs[r] = e
        finally:
            if ctx is not None:
                ctx.close()

    ts = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(JOIN_S)
        assert not t.is_alive(), "loopback rank hung"
    for e in errs:
        if e is not None:
            raise e
    return out


def build(dev, kind, ctx):
    if kind == "rmat":
        return dev.generate_rmat(12, 8, seed=3, ctx=ctx)
    if kind == "rmat_int":
        # integer weights through a CSR round trip of the R-MAT structure
        g = dev.generate_rmat(11, 8, seed=5, ctx=ctx)
        c = g.csr()
        # symmetric integer weights: w(u,v) = f(min, max)
        rows = np.repeat(np.arange(len(c["off"]) - 1), np.diff(c["off"]))
        lo, hi = np.minimum(rows, c["col"]), np.maximum(rows, c["col"])
        w = ((lo * 31 + hi * 17) % 5 + 1).astype(np.float32)
        return dev.Graph.from_csr(len(c["off"]) - 1, c["off"], c["col"], w, ctx=ctx)
    if kind == "lfr":
        g, _ = dev.generate_lfr(seed=2, ctx=ctx, n=20000, max_degree=120, min_community=20, max_community=400)
        return g
    if kind == "planted":
        g, _ = dev.generate_planted(4000, 40, 0.1, 0.002, seed=1, ctx=ctx)
        return g
    raise ValueError(kind)


def detect(dev, algo, g):
    if algo == "plp":
        cfg = dev.PlpConfig(randomize_order=True, seed=7)
        z, rep = dev.run_plp(g, cfg)
    elif algo == "plm":
        z, rep = dev.run_plm(g, dev.LouvainConfig(seed=7))
    elif algo == "plmr":
        z, rep = dev.run_plmr(g, dev.LouvainConfig(seed=7))
    elif algo == "epp":
        z, rep = dev.run_epp(g, dev.EnsembleConfig(ensemble_size=3, seed=7))
    else:
        raise ValueError(algo)
    return np.array(z), rep.modularity


def single(dev, kind, algo):
    ctx = dev.Context(0)
    try:
        return detect(dev, algo, build(dev, kind, ctx))
    finally:
        ctx.close()


CASES = [("rmat", "plp"), ("lfr", "plp"), ("rmat", "plm"), ("lfr", "plm"), ("planted", "plmr"),
         ("rmat_int", "plmr"), ("rmat", "epp"), ("lfr", "epp")]


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("layout", ["replicated", "rows"])
@pytest.mark.parametrize("kind,algo", CASES)
def test_sharded_equals_single(dev, G, layout, kind, algo):
    z1, q1 = single(dev, kind, algo)

    def fn(ctx, r):
        g = build(dev, kind, ctx)
        if layout == "rows":
            g = g.shard(ctx)
            lo, hi = g.owned_range
            assert 0 <= lo <= hi <= g.node_count()
        return detect(dev, algo, g)

    res = run_ranks(dev, G, fn)
    for r, (z, q) in enumerate(res):
        assert np.array_equal(z, z1), f"rank {r}: labels differ from the one-device run"
        assert q == pytest.approx(q1, rel=1e-9, abs=1e-12)


def test_sharded_real_weights_quality(dev):
    """fp32 weights: volumes are fp64 atomics (order-dependent even on one
    device), so only the labels' consistency across ranks and the quality
    are pinned."""
    def mk(ctx):
        return dev.generate_rmat(12, 8, weighted=True, seed=9, ctx=ctx)

    ctx = dev.Context(0)
    _, rep1 = dev.run_plmr(mk(ctx), dev.LouvainConfig(seed=3))
    ctx.close()
    res = run_ranks(dev, 2, lambda c, r: dev.run_plmr(mk(c).shard(c), dev.LouvainConfig(seed=3)))
    z0 = np.array(res[0][0])
    assert np.array_equal(z0, np.array(res[1][0]))
    assert abs(res[0][1].modularity - rep1.modularity) < 0.005


def test_shard_layout_and_quality(dev):
    """A row shard keeps only its rows; modularity and coarsening over the
    shards equal the whole graph's."""
    ctx0 = dev.Context(0)
    g1 = build(dev, "lfr", ctx0)
    z1, _ = dev.run_plm(g1, dev.LouvainConfig(seed=1))
    q1 = dev.modularity(g1, z1)
    full = g1.csr()
    coarse1 = dev.coarsen(g1, z1)[0].csr()

    def fn(ctx, r):
        g = build(dev, "lfr", ctx).shard(ctx)
        lo, hi = g.owned_range
        c = g.csr()
        deg = np.diff(c["off"])
        assert np.all(deg[:lo] == 0) and np.all(deg[hi:] == 0)
        assert np.array_equal(c["col"], full["col"][full["off"][lo]:full["off"][hi]])
        np.testing.assert_array_equal(c["vol"], full["vol"])
        q = dev.modularity(g, z1)
        cg = dev.coarsen(g, z1)[0].csr()
        return lo, hi, q, cg

    res = run_ranks(dev, 3, fn)
    bounds = [res[0][0]] + [r[1] for r in res]
    assert bounds[0] == 0 and bounds[-1] == g1.node_count()
    assert all(res[i][1] == res[i + 1][0] for i in range(2))
    assert list(bounds) == list(dev.shard_bounds(full["off"], 3))
    for _, _, q, cg in res:
        assert q == pytest.approx(q1, rel=1e-12)
        for key in ("off", "col", "w", "vol", "loop"):
            np.testing.assert_array_equal(cg[key], coarse1[key])
    ctx0.close()


def test_nccl_world_one(dev):
    """The NCCL transport (libnccl.so.2, loaded on first use) at world size 1:
    every sub-sweep still goes through ncclAllGather."""
    z1, q1 = single(dev, "lfr", "plm")
    ctx = dev.Context(0)
    try:
        ctx.attach_nccl(1, 0, dev.nccl_unique_id())
        assert ctx.world == (0, 1)
        z, q = detect(dev, "plm", build(dev, "lfr", ctx))
        assert np.array_equal(z, z1) and q == q1
        z, _ = detect(dev, "plp", build(dev, "lfr", ctx).shard(ctx))
        z2, _ = single(dev, "lfr", "plp")
        assert np.array_equal(z, z2)
    finally:
        ctx.close()


@pytest.mark.parametrize("layout", ["replicated", "rows"])
def test_sharded_tiny_graphs_more_ranks_than_nodes(dev, layout):
    """Ranks owning no nodes (G > n), isolated nodes and a self-loop."""
    cases = [(3, [(0, 1), (1, 2)]), (5, [(0, 1), (1, 2), (2, 0), (3, 3)]), (2, [(0, 1)])]
    for n, edges in cases:
        def mk(ctx):
            return dev.Graph.from_edges(n, edges, ctx=ctx)

        ctx0 = dev.Context(0)
        z1 = {a: detect(dev, a, mk(ctx0))[0] for a in ("plp", "plm", "plmr")}
        ctx0.close()

        def fn(ctx, r):
            g = mk(ctx)
            if layout == "rows":
                g = g.shard(ctx)
            return {a: detect(dev, a, g)[0] for a in ("plp", "plm", "plmr")}

        for res in run_ranks(dev, 4, fn):
            for a in z1:
                assert np.array_equal(res[a], z1[a]), (n, a)


def _info(g):
    return (g.node_count(), g.edge_count(), g.total_edge_weight(), g.max_degree, g.isolated)


@pytest.mark.parametrize("weighted", [False, True])
def test_rmat_chunked_builder(dev, monkeypatch, weighted):
    """The R-MAT builder in many row chunks (CD_BUILD_CHUNK_ENTRIES) gives the
    same CSR as the one-chunk build (which the oracle pins bit-exactly)."""
    ctx = dev.Context(0)
    try:
        ref = dev.generate_rmat(12, 8, weighted=weighted, seed=4, ctx=ctx).csr()
        for chunk in ("7000", "1"):
            monkeypatch.setenv("CD_BUILD_CHUNK_ENTRIES", chunk)
            c = dev.generate_rmat(12, 8, weighted=weighted, seed=4, ctx=ctx).csr()
            for key in ref:
                np.testing.assert_array_equal(c[key], ref[key], err_msg=f"{key} chunk={chunk}")
    finally:
        ctx.close()


@pytest.mark.parametrize("G", [2, 3])
def test_generated_rmat_shard(dev, monkeypatch, G):
    """cd_graph_generate_rmat_shard: every rank builds only its rows (in
    several chunks here); the rows, node state and graph totals equal the
    whole graph's, and PLM / PLP over the generated shards give the one-device
    labels."""
    monkeypatch.setenv("CD_BUILD_CHUNK_ENTRIES", "20000")
    ctx0 = dev.Context(0)
    g1 = dev.generate_rmat(13, 8, seed=6, ctx=ctx0)
    full, info1 = g1.csr(), _info(g1)
    zm, _ = dev.run_plm(g1, dev.LouvainConfig(seed=7))
    zp, _ = dev.run_plp(g1, dev.PlpConfig(randomize_order=True, seed=7))
    zm, zp = np.array(zm), np.array(zp)
    ctx0.close()

    def fn(ctx, r):
        g = dev.generate_rmat(13, 8, seed=6, ctx=ctx, shard=True)
        assert g.is_shard
        lo, hi = g.owned_range
        c = g.csr()
        deg = np.diff(c["off"])
        assert np.all(deg[:lo] == 0) and np.all(deg[hi:] == 0)
        assert np.array_equal(c["col"], full["col"][full["off"][lo]:full["off"][hi]])
        np.testing.assert_array_equal(c["vol"], full["vol"])
        assert _info(g) == info1
        z1 = np.array(dev.run_plm(g, dev.LouvainConfig(seed=7))[0])
        z2 = np.array(dev.run_plp(g, dev.PlpConfig(randomize_order=True, seed=7))[0])
        return lo, hi, z1, z2

    res = run_ranks(dev, G, fn)
    assert res[0][0] == 0 and res[-1][1] == info1[0]
    assert all(res[i][1] == res[i + 1][0] for i in range(G - 1))
    for _, _, z1, z2 in res:
        assert np.array_equal(z1, zm) and np.array_equal(z2, zp)


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("kind,algo", [("rmat", "plm"), ("lfr", "plm"), ("planted", "plmr"), ("rmat_int", "plmr"),
                                       ("rmat", "epp")])
def test_sharded_coarse_levels(dev, monkeypatch, G, kind, algo):
    """Coarse graphs too large to replicate stay row-sharded (C5): every
    rank sends each coarse-row owner its partial slab (all-to-all) and the
    owner merges them.  Forced at every level here; labels must equal the
    one-device run."""
    z1, q1 = single(dev, kind, algo)
    monkeypatch.setenv("CD_SHARD_COARSE_MIN_ENTRIES", "0")

    def fn(ctx, r):
        return detect(dev, algo, build(dev, kind, ctx).shard(ctx))

    for r, (z, q) in enumerate(run_ranks(dev, G, fn)):
        assert np.array_equal(z, z1), f"rank {r}: labels differ from the one-device run"
        assert q == pytest.approx(q1, rel=1e-9, abs=1e-12)


def test_sharded_coarse_graph_layout(dev, monkeypatch):
    """The sharded coarse graph of a row shard: each rank's rows equal the
    whole coarse graph's rows (as sets per row: detector-internal contraction
    leaves rows unsorted), node state and totals global."""
    ctx0 = dev.Context(0)
    g1 = build(dev, "lfr", ctx0)
    z1, _ = dev.run_plm(g1, dev.LouvainConfig(seed=1))
    cg1 = dev.coarsen(g1, z1)[0]
    full = cg1.csr()
    tot1 = (cg1.edge_count(), cg1.total_edge_weight(), cg1.max_degree, cg1.isolated)
    ctx0.close()
    monkeypatch.setenv("CD_SHARD_COARSE_MIN_ENTRIES", "0")

    def fn(ctx, r):
        cg = dev.coarsen(build(dev, "lfr", ctx).shard(ctx), z1)[0]
        assert cg.is_shard
        lo, hi = cg.owned_range
        c = cg.csr()
        deg = np.diff(c["off"])
        assert np.all(deg[:lo] == 0) and np.all(deg[hi:] == 0)
        np.testing.assert_array_equal(c["vol"], full["vol"])
        assert (cg.edge_count(), cg.total_edge_weight(), cg.max_degree, cg.isolated) == tot1
        for u in range(lo, hi):
            a = slice(c["off"][u], c["off"][u + 1])
            b = slice(full["off"][u], full["off"][u + 1])
            assert np.array_equal(c["col"][a], full["col"][b])  # the API contraction is sorted
            np.testing.assert_array_equal(c["w"][a], full["w"][b])
        return lo, hi

    res = run_ranks(dev, 3, fn)
    assert res[0][0] == 0 and res[-1][1] == full["off"].shape[0] - 1
    assert all(res[i][1] == res[i + 1][0] for i in range(2))


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("kind", ["rmat", "rmat_int", "planted"])
def test_row_shard_from_own_rows(dev, G, kind):
    """cd_graph_from_csr_rows: every rank uploads the offsets and only its own
    rows (bench.py's multi-GPU e2e) and gets the same row shard as cutting
    the whole graph (cd_graph_shard): layout, node state and totals, and the
    same labels as one device."""
    ctx0 = dev.Context(0)
    g1 = build(dev, kind, ctx0)
    full = g1.csr()
    n, m, total = g1.node_count(), g1.edge_count(), g1.total_edge_weight()
    z1, _ = detect(dev, "plm", g1)
    p1, _ = detect(dev, "plp", g1)
    ctx0.close()
    bounds = dev.shard_bounds(full["off"], G)

    def fn(ctx, r):
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        e0, e1 = int(full["off"][lo]), int(full["off"][hi])
        w = None if full["w"] is None else full["w"][e0:e1]
        g = dev.Graph.from_csr_rows(n, full["off"], lo, hi, full["col"][e0:e1], w, ctx=ctx)
        ref = build(dev, kind, ctx).shard(ctx)
        a, b = g.csr(), ref.csr()
        for key in ("off", "col", "vol", "loop"):
            np.testing.assert_array_equal(a[key], b[key])
        assert g.owned_range == ref.owned_range == (lo, hi)
        assert (g.edge_count(), g.total_edge_weight()) == (m, total)
        return detect(dev, "plm", g)[0], detect(dev, "plp", g)[0]

    for z, p in run_ranks(dev, G, fn):
        assert np.array_equal(z, z1) and np.array_equal(p, p1)


@pytest.mark.parametrize("weighted", [False, True])
def test_row_shard_from_own_rows_chunked(dev, weighted):
    """Row shards of at least 2^22 entries take the chunked upload (each
    chunk checked while the next one copies): same shard as the cut one, same
    labels as one device, and a defect inside a later chunk is an input error."""
    G = 2
    ctx0 = dev.Context(0)
    g1 = dev.generate_rmat(19, 16, weighted=weighted, seed=4, ctx=ctx0)
    full = g1.csr()
    n, m, total = g1.node_count(), g1.edge_count(), g1.total_edge_weight()
    p1, _ = detect(dev, "plp", g1)
    ctx0.close()
    bounds = dev.shard_bounds(full["off"], G)
    assert all(int(full["off"][bounds[r + 1]] - full["off"][bounds[r]]) >= (1 << 22) for r in range(G))

    def fn(ctx, r):
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        e0, e1 = int(full["off"][lo]), int(full["off"][hi])
        w = None if full["w"] is None else full["w"][e0:e1]
        g = dev.Graph.from_csr_rows(n, full["off"], lo, hi, full["col"][e0:e1], w, ctx=ctx)
        ref = dev.generate_rmat(19, 16, weighted=weighted, seed=4, ctx=ctx).shard(ctx)
        a, b = g.csr(), ref.csr()
        for key in ("off", "col", "vol", "loop"):
            np.testing.assert_array_equal(a[key], b[key])
        assert (g.edge_count(), g.total_edge_weight()) == (m, total)
        return detect(dev, "plp", g)[0]

    for p in run_ranks(dev, G, fn):
        assert np.array_equal(p, p1)
    # a neighbour out of range inside a later chunk (world size 1: the one rank's rows
    # are the whole graph)
    ctx = dev.Context(0)
    try:
        bad = full["col"].copy()
        bad[2 * (1 << 21) + 99] = n
        with pytest.raises(dev.InputError, match="malformed CSR"):
            dev.Graph.from_csr_rows(n, full["off"], 0, n, bad, full["w"], ctx=ctx)
    finally:
        ctx.close()


def test_row_shard_from_own_rows_checks_range(dev):
    """Every rank must pass exactly its cd_shard_bounds range (checked
    before any collective, so a wrong range fails on each rank alone)."""
    ctx0 = dev.Context(0)
    full = build(dev, "rmat", ctx0).csr()
    ctx0.close()
    n = len(full["off"]) - 1
    bounds = dev.shard_bounds(full["off"], 2)

    def fn(ctx, r):
        lo, hi = int(bounds[r]) + 1, int(bounds[r + 1])  # one row short
        e0, e1 = int(full["off"][lo]), int(full["off"][hi])
        with pytest.raises(dev.InvalidArgument, match="not this rank's shard range"):
            dev.Graph.from_csr_rows(n, full["off"], lo, hi, full["col"][e0:e1], ctx=ctx)
        return True

    assert all(run_ranks(dev, 2, fn))
