"""Text ingest throughput: device readers vs the reference's io::read_metis /
read_edge_list (oracle/_ref, host) on the same bytes.

    python tools/ingest_bench.py [--scale 20]

Writes an R-MAT graph (device generator) as METIS and as an edge list with
sparse 40-bit ids, then times: reference read (file -> Graph), device read
from host bytes (H2D + parse + CSR build), device read from device-resident
bytes.  Prints one line per format.
"""
import argparse
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1304_4453_b200 as P  # noqa: E402


def metis_bytes(c):
    n = len(c["off"]) - 1
    rows = np.repeat(np.arange(n), np.diff(c["off"]))
    m = int((c["col"] >= rows).sum())
    col1 = (c["col"] + 1).astype(str)
    parts = [f"{n} {m}"]
    for u in range(n):
        parts.append(" ".join(col1[c["off"][u]:c["off"][u + 1]]))
    return ("\n".join(parts) + "\n").encode()


def edges_bytes(c, rng):
    n = len(c["off"]) - 1
    rows = np.repeat(np.arange(n), np.diff(c["off"]))
    up = c["col"] > rows
    ids = np.unique(rng.integers(0, 1 << 40, size=2 * n, dtype=np.uint64))[:n]
    u, v = ids[rows[up]].astype(str), ids[c["col"][up]].astype(str)
    return ("\n".join(np.char.add(np.char.add(u, " "), v)) + "\n").encode()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    ctx = P.Context(0)
    g = P.generate_rmat(a.scale, 16, seed=1, ctx=ctx)
    c = g.csr()
    rng = np.random.default_rng(0)
    from oracle import oracle as O
    for kind, data in (("metis", metis_bytes(c)), ("edges", edges_bytes(c, rng))):
        with tempfile.NamedTemporaryFile(suffix="." + kind, delete=False) as f:
            f.write(data)
            path = f.name
        res = {"format": kind, "bytes": len(data), "m": g.edge_count()}
        if O.ref_available():
            t0 = time.perf_counter()
            if kind == "metis":
                rg = O.RefGraph.read_metis(path)
            else:
                rg, _ = O.RefGraph.read_edge_list(path, max_ids=len(c["off"]))
            res["ref_s"] = time.perf_counter() - t0
            del rg
        read = P.read_metis if kind == "metis" else P.read_edge_list
        dev_bytes = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
        for label, src in (("dev_from_host_s", data), ("dev_from_hbm_s", dev_bytes)):
            ts = []
            for _ in range(a.reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                g2 = read(src, ctx=ctx)
                ctx.synchronize()
                ts.append(time.perf_counter() - t0)
                assert g2.edge_count() == g.edge_count()
                del g2
            res[label] = min(ts)
        res["dev_GB_per_s"] = len(data) / res["dev_from_hbm_s"] / 1e9
        if "ref_s" in res:
            res["speedup_vs_ref"] = res["ref_s"] / res["dev_from_host_s"]
        os.unlink(path)
        print(res, flush=True)


if __name__ == "__main__":
    main()
