"""The sharded protocol across processes, on the CPU.

Two ranks talk over torch.distributed (gloo, 127.0.0.1).  Each owns the node
range the product's cd_shard_bounds assigns (host function of the C ABI, no
GPU needed), evaluates only its own nodes per sub-sweep (oracle restatement of
the device decision rule: cdo_plp_subsweep / cdo_move_subsweep), allgathers
the move lists and applies all of them in rank order -- exactly what the
device Sweeper does with NCCL.  The result must equal the one-process
bucketed drivers bit for bit.  The oracle is the checker here; the product
path of the same protocol is tests/test_gpu_shard.py.
"""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graph(kind):
    from oracle import oracle as O
    if kind == "planted":
        g, _ = O.generate_planted(3000, 30, 0.08, 0.003, 5)
        return g
    return O.generate_rmat(11, 8, seed=4)


def _bounds(off, G):
    import paper_1304_4453_b200 as P
    return P.shard_bounds(off, G)


def _apply_activation(g, us, active):
    for u in us:
        active[g.col[g.off[u]:g.off[u + 1]]] = 1


def plp_sharded(g, rank, G, allgather, seed=3, buckets=4, max_iterations=100):
    from oracle import oracle as O
    b = _bounds(g.off, G)
    lo, hi = int(b[rank]), int(b[rank + 1])
    n = g.n
    labels = np.arange(n, dtype=np.int32)
    active = np.ones(n, np.uint8)
    theta = max(1, n // 100000)
    updated, it = n, 0
    trace = []
    while updated > theta and it < max_iterations:
        updated = 0
        key = O.bucket_key(seed, it)
        for bk in range(buckets):
            mu, ml = O.plp_subsweep(g, labels, active, key, bk, buckets, lo, hi)
            for ru, rl in allgather((mu, ml)):  # rank order
                labels[ru] = rl
                _apply_activation(g, ru, active)
                updated += len(ru)
        trace.append(updated)
        it += 1
    return labels, trace


def move_phase_sharded(g, rank, G, allgather, seed=3, buckets=4, max_move_iterations=32, move_tol=1e-3,
                       move_stall=0.95, move_qtol=2e-3):
    from oracle import oracle as O
    b = _bounds(g.off, G)
    lo, hi = int(b[rank]), int(b[rank + 1])
    n = g.n
    z = np.arange(n, dtype=np.int32)
    vols = O.community_volumes(g, z, n)
    csize = np.ones(n, np.int32)
    active = np.ones(n, np.uint8)  # pruning (default on)
    theta = max(n // 100000, int(move_tol * n))
    hist = [-1, -1]
    cum = 0
    for p in range(max_move_iterations):
        key = O.bucket_key(seed, p)  # salt 0 = level 0, first phase
        moved = 0
        pass_fx = 0
        for bk in range(buckets):
            mu, ml, gfx = O.move_subsweep(g, z, vols, csize, active, key, bk, lo, hi, seed=seed, buckets=buckets)
            gathered = allgather((mu, ml, gfx))
            pass_fx += sum(x[2] for x in gathered)
            for ru, rl, _ in gathered:
                for u, d in zip(ru.tolist(), rl.tolist()):
                    c = z[u]
                    vols[c] -= g.vol[u]
                    vols[d] += g.vol[u]
                    csize[c] -= 1
                    csize[d] += 1
                    z[u] = d
                moved += len(ru)
            O.activate(g, np.concatenate([ru for ru, _, _ in gathered]), active)
        if moved == 0 or moved <= theta:
            break
        if move_stall > 0 and p >= 8 and moved > move_stall * hist[0]:
            break
        cum += pass_fx
        if move_qtol > 0 and float(pass_fx) <= move_qtol * float(cum):
            break
        hist = [hist[1], moved]
    return z


def _worker(rank, port, kind, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)

        def allgather(obj):
            out = [None] * WORLD
            dist.all_gather_object(out, obj)
            return out

        g = _graph(kind)
        labels, trace = plp_sharded(g, rank, WORLD, allgather)
        z = move_phase_sharded(g, rank, WORLD, allgather)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, labels, trace, z, None))
    except BaseException as e:  # noqa: BLE001 -- reported to the parent
        q.put((rank, None, None, None, repr(e)))


@pytest.mark.parametrize("kind", ["planted", "rmat"])
def test_gloo_two_ranks_match_single_process(kind):
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, kind, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(WORLD):
        r, labels, trace, z, err = q.get(timeout=240)
        assert err is None, f"rank {r}: {err}"
        res[r] = (labels, trace, z)
    for p in procs:
        p.join(60)
    g = _graph(kind)
    ref_labels, ref_trace = O.plp_bucketed(g, seed=3, buckets=4)
    ref_z, _ = O.move_phase_bucketed(g, np.arange(g.n), salt=0, seed=3, buckets=4)
    for r in range(WORLD):
        labels, trace, z = res[r]
        assert np.array_equal(labels, ref_labels)
        assert list(trace) == list(ref_trace)
        assert np.array_equal(z, ref_z)


def _row_shard(g, lo, hi):
    """The oracle CSR holding only rows [lo, hi) (global column ids)."""
    from oracle import oracle as O
    idx = np.arange(g.n + 1)
    off = np.where(idx <= lo, 0, np.where(idx >= hi, g.off[hi] - g.off[lo], g.off[np.minimum(idx, g.n)] - g.off[lo]))
    return O.from_csr(g.n, off, g.col[g.off[lo]:g.off[hi]], g.w[g.off[lo]:g.off[hi]])


def coarse_shard_sharded(g, zc, rank, G, allgather):
    """The sharded contraction (csrc/shard.cu coarse_shard_from_partials):
    partial coarse graph of this rank's rows; coarse-row owners from the
    summed partial row lengths (cd_shard_bounds); every rank sends each owner
    its slab; the owner merges (sum by label, rows ascending)."""
    from oracle import oracle as O
    b = _bounds(g.off, G)
    part = O.coarsen(_row_shard(g, int(b[rank]), int(b[rank + 1])), zc)
    nc = part.n
    lens = sum(allgather(np.diff(part.off)))
    cb = _bounds(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64), G)
    # slabs for every owner (all_gather_object stands in for the all-to-all)
    slabs = allgather([(part.off[cb[d]:cb[d + 1] + 1] - part.off[cb[d]],
                        part.col[part.off[cb[d]]:part.off[cb[d + 1]]],
                        part.w[part.off[cb[d]]:part.off[cb[d + 1]]]) for d in range(G)])
    lo, hi = int(cb[rank]), int(cb[rank + 1])
    rows = []
    for c in range(lo, hi):
        acc = {}
        for s in range(G):
            roff, col, w = slabs[s][rank]
            i = c - lo
            for k, x in zip(col[roff[i]:roff[i + 1]], w[roff[i]:roff[i + 1]]):
                acc[int(k)] = acc.get(int(k), 0.0) + float(x)
        rows.append(sorted(acc.items()))
    return lo, hi, nc, rows


def _worker_coarse(rank, port, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)

        def allgather(obj):
            out = [None] * WORLD
            dist.all_gather_object(out, obj)
            return out

        from oracle import oracle as O
        g = O.generate_rmat(10, 8, seed=4)
        z, _ = O.move_phase_bucketed(g, np.arange(g.n), salt=0, seed=3, buckets=4)
        zc, _ = O.compact(z)
        out = coarse_shard_sharded(g, zc, rank, WORLD, allgather)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except BaseException as e:  # noqa: BLE001 -- reported to the parent
        q.put((rank, None, repr(e)))


def test_gloo_sharded_contraction_matches_whole():
    """Two processes build the sharded coarse graph; the owners' rows, put
    together, are the whole graph's contraction (oracle coarsen)."""
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_coarse, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(WORLD):
        r, out, err = q.get(timeout=240)
        assert err is None, f"rank {r}: {err}"
        res[r] = out
    for p in procs:
        p.join(60)
    g = O.generate_rmat(10, 8, seed=4)
    z, _ = O.move_phase_bucketed(g, np.arange(g.n), salt=0, seed=3, buckets=4)
    zc, _ = O.compact(z)
    cg = O.coarsen(g, zc)
    assert res[0][0] == 0 and res[WORLD - 1][1] == cg.n and res[0][1] == res[1][0]
    for r in range(WORLD):
        lo, hi, nc, rows = res[r]
        assert nc == cg.n
        for c, row in zip(range(lo, hi), rows):
            seg = slice(cg.off[c], cg.off[c + 1])
            assert [k for k, _ in row] == cg.col[seg].tolist()
            np.testing.assert_allclose([x for _, x in row], cg.w[seg], rtol=1e-12)


def test_shard_bounds_host():
    """cd_shard_bounds: first node whose offset reaches D*r/G (no GPU)."""
    import paper_1304_4453_b200 as P
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 1000):
        deg = rng.integers(0, 50, size=n)
        deg[rng.random(n) < 0.1] = 0
        off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        D = int(off[-1])
        for G in (1, 2, 3, 8):
            b = P.shard_bounds(off, G)
            exp = [0] + [int(np.searchsorted(off[:n], D * r // G, side="left")) for r in range(1, G)] + [n]
            assert list(b) == exp
            assert all(b[i] <= b[i + 1] for i in range(G))
