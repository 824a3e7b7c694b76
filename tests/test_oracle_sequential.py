"""The oracle's sequential move phase (one worker, H/louvain.hpp:65-141) and its
move log (the MoveObserver's arguments, :60, :127-128) pinned to the
reference itself (oracle/_ref, move_phase with an observer).

The reference's own check of this path is tests/test_louvain.cpp:85-98 and
acceptance criterion 6 (tests/acceptance.cpp:164-176): with one worker every
observed move strictly raises modularity."""
import numpy as np
import pytest

from conftest import rand_edges


def _graph(oracle, seed, n, p, kind, loop_p=0.1):
    rng = np.random.default_rng(seed)
    eu, ev, ew = rand_edges(rng, n, p, kind, loop_p)
    return oracle.from_arrays(n, eu, ev, ew)


@pytest.mark.parametrize("kind", ["unit", "int", "real"])
def test_sequential_move_phase_matches_reference(oracle, ref, kind):
    for i in range(12):
        og = _graph(oracle, 500 + i, 8 + 7 * i, 0.3 if i < 6 else 0.08, kind)
        rg = ref.RefGraph.from_csr(og)
        z0 = np.arange(og.n, dtype=np.int32)
        zr, chr_, moves_r, _ = rg.move_phase_log(z0, max_move_iterations=32, workers=1)
        zo, cho, moves_o = oracle.move_phase_sequential(og, z0, max_move_iterations=32)
        assert cho == chr_
        assert np.array_equal(zo, zr), f"case {i}"
        assert moves_o == moves_r, f"case {i}"


def test_sequential_moves_strictly_raise_modularity(oracle, ref):
    # tests/test_louvain.cpp:85-98 on the reference; the oracle's log replays it
    for i in range(10):
        og = _graph(oracle, 900 + i, 8 + i % 12, 0.35, "unit")
        z = np.arange(og.n, dtype=np.int32)
        _, _, moves = oracle.move_phase_sequential(og, z)
        last = oracle.modularity(og, z, ub=og.n)
        for u, c, d, gain in moves:
            assert z[u] == c and gain > 0
            z[u] = d
            q = oracle.modularity(og, z, ub=og.n)
            assert q > last
            last = q


def test_sequential_pass_cap_and_labels(oracle, ref):
    og = _graph(oracle, 77, 40, 0.2, "int")
    rg = ref.RefGraph.from_csr(og)
    z0 = np.arange(og.n, dtype=np.int32)
    for cap in (0, 1, 2):
        zr, chr_, mr, _ = rg.move_phase_log(z0, max_move_iterations=cap, workers=1)
        zo, cho, mo = oracle.move_phase_sequential(og, z0, max_move_iterations=cap)
        assert (cho, mo) == (chr_, mr) and np.array_equal(zo, zr)
    # labels outside [0, ub) -> out_of_range
    with pytest.raises(oracle.OracleOutOfRange):
        oracle.move_phase_sequential(og, np.full(og.n, 50, np.int32), ub=40)
