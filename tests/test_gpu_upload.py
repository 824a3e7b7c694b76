"""cd_graph_from_csr with host arrays of at least UPLOAD_MIN_ENTRIES (2^22)
entries: the columns are copied in chunks (upload_chunk(D): a power of two near
D / 8 within [2^21, 2^25], so 2^25 is a chunk boundary of the big fixtures),
each validated while the next one copies (graph_upload_validate).  The graph must equal the device-built one, and a
defect in any chunk -- or right at a chunk boundary -- must raise the same
input error as the unchunked path (H/graph.hpp:48-81 semantics)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CHUNK = 1 << 25


@pytest.fixture(scope="module")
def big(dev, ctx):
    g = dev.generate_rmat(21, 16, weighted=True, seed=2)  # ~63M entries: two chunks
    c = g.csr()
    assert len(c["col"]) > CHUNK
    return g, c


def test_chunked_upload_equals_device_graph(dev, big):
    g, c = big
    h = dev.Graph.from_csr(g.node_count(), c["off"], c["col"], c["w"])
    d = h.csr()
    assert np.array_equal(d["off"], c["off"]) and np.array_equal(d["col"], c["col"])
    assert np.array_equal(d["w"], c["w"])
    np.testing.assert_array_equal(d["vol"], c["vol"])
    assert h.edge_count() == g.edge_count() and h.total_edge_weight() == g.total_edge_weight()


@pytest.mark.parametrize("where", ["second_chunk", "boundary"])
def test_chunked_upload_rejects_unsorted_row(dev, big, where):
    g, c = big
    off, col = c["off"], c["col"].copy()
    target = CHUNK + 12345 if where == "second_chunk" else CHUNK
    u = int(np.searchsorted(off, target, side="right") - 1)
    while off[u + 1] - off[u] < 2:  # a row with two entries at or after the target
        u += 1
    i = max(int(off[u]) + 1, target) if target < off[u + 1] else int(off[u]) + 1
    col[i - 1], col[i] = col[i], col[i - 1]  # breaks the strictly ascending order
    with pytest.raises(dev.InputError, match="malformed CSR"):
        dev.Graph.from_csr(g.node_count(), off, col, c["w"])


def test_chunked_upload_rejects_out_of_range(dev, big):
    g, c = big
    col = c["col"].copy()
    col[-1] = g.node_count()  # the last chunk
    with pytest.raises(dev.InputError, match="malformed CSR"):
        dev.Graph.from_csr(g.node_count(), c["off"], col, c["w"])


@pytest.fixture(scope="module")
def big_unweighted(dev, ctx):
    """An unweighted graph above two chunks with self-loops scattered over
    every chunk (built on the device, so its node state comes from
    graph_finalize)."""
    g = dev.generate_rmat(21, 16, weighted=False, seed=3)
    c = g.csr()
    n = g.node_count()
    deg = np.diff(c["off"])
    u = np.repeat(np.arange(n, dtype=np.int64), deg)
    v = c["col"].astype(np.int64)
    keep = u <= v
    loops = np.arange(0, n, 997, dtype=np.int64)
    gl = dev.Graph.from_edges(n, (np.concatenate([u[keep], loops]), np.concatenate([v[keep], loops])))
    cl = gl.csr()
    assert len(cl["col"]) > CHUNK and cl["loop"].sum() == len(loops)
    return gl, cl


def test_chunked_upload_unweighted_finalized_during_copy(dev, big_unweighted):
    """Unweighted chunks also count self-loops and upper entries, and the
    degree tiers are built from the offsets while the columns copy: node
    state, totals and a PLP run equal the device-built graph's."""
    g, c = big_unweighted
    h = dev.Graph.from_csr(g.node_count(), c["off"], c["col"])
    d = h.csr()
    assert np.array_equal(d["col"], c["col"])
    np.testing.assert_array_equal(d["vol"], c["vol"])
    np.testing.assert_array_equal(d["loop"], c["loop"])
    assert (h.edge_count(), h.total_edge_weight(), h.max_degree, h.isolated) == \
        (g.edge_count(), g.total_edge_weight(), g.max_degree, g.isolated)
    la, _ = dev.run_plp(h, dev.PlpConfig(seed=1))
    lb, _ = dev.run_plp(g, dev.PlpConfig(seed=1))
    assert np.array_equal(la, lb)


def test_chunked_upload_unweighted_rejects(dev, big_unweighted):
    g, c = big_unweighted
    col = c["col"].copy()
    col[CHUNK + 7] = g.node_count() + 5  # second chunk
    with pytest.raises(dev.InputError, match="malformed CSR"):
        dev.Graph.from_csr(g.node_count(), c["off"], col)
    off = c["off"].copy()
    off[10] = off[11] + 1  # descending offsets: rejected before the tiers are built
    with pytest.raises(dev.InputError, match="malformed CSR"):
        dev.Graph.from_csr(g.node_count(), off, c["col"])


# ---- mid-size graphs: chunks of 2^21 entries (csrc/graph.cuh upload_chunk) -------
SMALL_CHUNK = 1 << 21


@pytest.fixture(scope="module", params=[False, True], ids=["unweighted", "weighted"])
def mid(request, dev, ctx):
    g = dev.generate_rmat(18, 16, weighted=request.param, seed=5)  # ~8M entries: four chunks of 2^21
    c = g.csr()
    assert (1 << 22) <= len(c["col"]) <= 8 * SMALL_CHUNK
    return g, c


def test_mid_size_chunked_upload_equals_device_graph(dev, mid):
    g, c = mid
    h = dev.Graph.from_csr(g.node_count(), c["off"], c["col"], c["w"])
    d = h.csr()
    assert np.array_equal(d["off"], c["off"]) and np.array_equal(d["col"], c["col"])
    if c["w"] is not None:
        assert np.array_equal(d["w"], c["w"])
    np.testing.assert_array_equal(d["vol"], c["vol"])
    np.testing.assert_array_equal(d["loop"], c["loop"])
    assert (h.edge_count(), h.total_edge_weight(), h.max_degree, h.isolated) == \
        (g.edge_count(), g.total_edge_weight(), g.max_degree, g.isolated)
    la, _ = dev.run_plm(h)
    lb, _ = dev.run_plm(g)
    assert np.array_equal(la, lb)


@pytest.mark.parametrize("where", ["boundary", "third_chunk", "last_entry"])
def test_mid_size_chunked_upload_rejects(dev, mid, where):
    g, c = mid
    off, col = c["off"], c["col"].copy()
    if where == "last_entry":
        col[-1] = g.node_count()
    else:
        target = SMALL_CHUNK if where == "boundary" else 2 * SMALL_CHUNK + 4321
        u = int(np.searchsorted(off, target, side="right") - 1)
        while off[u + 1] - off[u] < 2:
            u += 1
        i = max(int(off[u]) + 1, target) if target < off[u + 1] else int(off[u]) + 1
        col[i - 1], col[i] = col[i], col[i - 1]
    with pytest.raises(dev.InputError, match="malformed CSR"):
        dev.Graph.from_csr(g.node_count(), off, col, c["w"])
