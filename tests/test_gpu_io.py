"""Device text readers (cd_graph_read_metis / cd_graph_read_edge_list /
cd_graph_load_*) against the reader oracle (oracle/io_oracle.py, itself pinned
to the reference by tests/test_io_oracle.py): identical CSR structure, weights
equal after the fp32 storage rounding, identical original ids, and the same
error class for every malformed file of the corpus.  Plus round trips of
device-generated graphs at ~1M entries through text."""
import numpy as np
import pytest

from io_cases import cases, category

pytestmark = pytest.mark.gpu


def _dev_read(dev, kind, text, merge):
    if kind == "metis":
        return dev.read_metis(text)
    return dev.read_edge_list(text, merge_duplicates=merge)


@pytest.mark.parametrize("name,kind,text,merge", cases(), ids=[c[0] for c in cases()])
def test_reader_matches_oracle(dev, ctx, name, kind, text, merge):
    from oracle import io_oracle as IO
    ora_err = None
    try:
        if kind == "metis":
            og, weighted = IO.read_metis(text, "<metis>")
            oids = None
        else:
            og, oids, weighted = IO.read_edge_list(text, merge, "<edge list>")
    except IO.InputError as e:
        ora_err = str(e)
    if ora_err is not None:
        with pytest.raises(dev.InputError) as ei:
            _dev_read(dev, kind, text, merge)
        assert category(str(ei.value)) == category(ora_err), (str(ei.value), ora_err)
        return
    g = _dev_read(dev, kind, text, merge)
    c = g.csr()
    assert g.node_count() == og.n and g.edge_count() == og.m
    np.testing.assert_array_equal(c["off"], og.off)
    np.testing.assert_array_equal(c["col"], og.col)
    w = c["w"] if c["w"] is not None else np.ones(len(c["col"]), np.float32)
    np.testing.assert_array_equal(w, og.w.astype(np.float32))
    if kind == "edges":
        np.testing.assert_array_equal(g.original_ids(), oids)


@pytest.mark.parametrize("kind,text", [
    ("metis", b"2 1 1\n2 1e-50\n1 1e-50\n"), ("metis", b"2 1 1\n2 1e300\n1 1e300\n"),
    ("edges", b"0 1 1e-50\n"), ("edges", b"0 1 1e300\n")])
def test_weight_not_fp32_representable(dev, ctx, kind, text):
    """Weights are stored as fp32: a positive weight that would round to 0 or
    overflow to inf is rejected with its line (the reference keeps fp64)."""
    with pytest.raises(dev.InputError, match="not a positive finite fp32 value"):
        _dev_read(dev, kind, text, False)


def test_load_from_path_messages(dev, tmp_path):
    """cd_graph_load_*: the path prefixes messages like the reference's."""
    p = tmp_path / "g.metis"
    p.write_bytes(b"2 1\n2\n1\n")
    g = dev.read_metis(str(p))
    assert g.edge_count() == 1
    bad = tmp_path / "bad.metis"
    bad.write_bytes(b"2 1\n3\n1\n")
    with pytest.raises(dev.InputError, match=str(bad) + ":2: neighbor id 3 out of range"):
        dev.read_metis(str(bad))
    with pytest.raises(dev.InputError, match="cannot open"):
        dev.read_metis(str(tmp_path / "missing.metis"))
    e = tmp_path / "g.edges"
    e.write_bytes(b"100 200\n200 300 # c\n")
    g = dev.read_edge_list(str(e))
    assert list(g.original_ids()) == [100, 200, 300]


def _write_metis(c, weighted):
    n = len(c["off"]) - 1
    m = int(((c["col"] >= np.repeat(np.arange(n), np.diff(c["off"]))).sum()))
    lines = [f"{n} {m}" + (" 1" if weighted else "")]
    col1 = (c["col"] + 1).astype(str)
    wts = c["w"].astype(np.float64).astype(str) if weighted else None
    for u in range(n):
        s, e = c["off"][u], c["off"][u + 1]
        if weighted:
            lines.append(" ".join(f"{a} {b}" for a, b in zip(col1[s:e], wts[s:e])))
        else:
            lines.append(" ".join(col1[s:e]))
    return ("\n".join(lines) + "\n").encode()


@pytest.mark.parametrize("weighted", [False, True])
def test_metis_round_trip_large(dev, ctx, weighted):
    g = dev.generate_rmat(15, 16, weighted=weighted, seed=11)
    c = g.csr()
    g2 = dev.read_metis(_write_metis(c, weighted))
    c2 = g2.csr()
    np.testing.assert_array_equal(c2["off"], c["off"])
    np.testing.assert_array_equal(c2["col"], c["col"])
    if weighted:
        np.testing.assert_array_equal(c2["w"], c["w"])  # repr() of fp32 values round-trips
    assert g2.edge_count() == g.edge_count()


def test_edge_list_round_trip_large(dev, ctx):
    g = dev.generate_rmat(15, 16, seed=12)
    c = g.csr()
    n = g.node_count()
    rows = np.repeat(np.arange(n), np.diff(c["off"]))
    up = c["col"] > rows
    rng = np.random.default_rng(3)
    ids = np.unique(rng.integers(0, 1 << 40, size=2 * n, dtype=np.uint64))
    assert len(ids) >= n
    ids = np.sort(rng.permutation(ids)[:n])
    u, v = ids[rows[up]], ids[c["col"][up]]
    order = rng.permutation(len(u))
    text = "\n".join(f"{a} {b}" for a, b in zip(u[order], v[order])).encode()
    g2 = dev.read_edge_list(text)
    used = np.unique(np.concatenate([rows[up], c["col"][up]]))
    np.testing.assert_array_equal(g2.original_ids(), ids[used])
    assert g2.edge_count() == g.edge_count()
    # structure: the subgraph on used nodes, relabelled densely in id order
    remap = -np.ones(n, np.int64)
    remap[used] = np.arange(len(used))
    c2 = g2.csr()
    deg = np.diff(c["off"])[used]
    np.testing.assert_array_equal(np.diff(c2["off"]), deg)
    np.testing.assert_array_equal(c2["col"], remap[c["col"][np.isin(rows, used)]])
