"""Pins the reader oracle (oracle/io_oracle.py) to the unmodified reference
readers (oracle/_ref: io::read_metis / io::read_edge_list, H/io.hpp) on the
whole corpus of tests/io_cases.py: same CSR (offsets, columns, fp64 weights,
m) and original ids, or the same error message."""
import numpy as np
import pytest

from io_cases import cases


def _ref_read(ref, kind, path, merge):
    if kind == "metis":
        return ref.RefGraph.read_metis(path), None
    return ref.RefGraph.read_edge_list(path, merge)


@pytest.mark.parametrize("name,kind,text,merge", cases(), ids=[c[0] for c in cases()])
def test_reader_oracle_matches_reference(ref, tmp_path, name, kind, text, merge):
    from oracle import io_oracle as IO
    path = str(tmp_path / f"{name}.txt")
    with open(path, "wb") as f:
        f.write(text)
    ref_err = ora_err = None
    try:
        rg, rids = _ref_read(ref, kind, path, merge)
    except ref.OracleInputError as e:
        ref_err = str(e).split(": ", 1)[1]  # strip the code prefix
    try:
        if kind == "metis":
            og, _ = IO.read_metis(text, path)
            oids = None
        else:
            og, oids, _ = IO.read_edge_list(text, merge, path)
    except IO.InputError as e:
        ora_err = str(e)
    if ref_err is not None or ora_err is not None:
        assert ref_err == ora_err, (ref_err, ora_err)
        assert name.startswith("err") or "_err_" in name
        return
    assert not (name.startswith("err") or "_err_" in name)
    c = rg.csr()
    assert c.n == og.n and c.m == og.m
    np.testing.assert_array_equal(c.off, og.off)
    np.testing.assert_array_equal(c.col, og.col)
    np.testing.assert_array_equal(c.w, og.w)
    if kind == "edges":
        np.testing.assert_array_equal(rids, oids)
