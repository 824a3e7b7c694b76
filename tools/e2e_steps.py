"""Per-step anatomy of bench.py's end-to-end leg (one B200): N consecutive e2e
steps, each split by CUDA events on the library stream into cd_graph_from_csr
(H2D + validation + finalize + tiers) and the detector (+ D2H of the labels),
with the host wall time beside it.  Shows whether a slow e2e mean is one stalled
step or a slow link.

    python tools/e2e_steps.py [--workload c3_rmat24_plp] [--steps 12]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1304_4453_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_rmat24_plp", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--steps", type=int, default=12)
    a = ap.parse_args()
    wl = bench.WORKLOADS[a.workload]
    ctx = P.Context(0)
    g = bench.make_device_graph(P, ctx, wl)
    n = g.node_count()
    c = g.csr()
    del g
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
    t_off, t_col = pin(c["off"]), pin(c["col"])
    t_w = pin(c["w"]) if c["w"] is not None else None
    h_out = torch.empty(n, dtype=torch.int32).pin_memory().numpy()
    stream = torch.cuda.ExternalStream(ctx.stream)
    rows = []
    for i in range(a.steps + 1):
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        h0 = time.perf_counter()
        ev[0].record(stream)
        gh = P.Graph.from_csr(n, t_off.numpy(), t_col.numpy(), None if t_w is None else t_w.numpy(), ctx=ctx)
        h1 = time.perf_counter()
        ev[1].record(stream)
        bench.run_device(P, gh, wl["algo"], h_out, report=False)
        ev[2].record(stream)
        ev[2].synchronize()
        h2 = time.perf_counter()
        del gh
        h3 = time.perf_counter()
        if i:
            rows.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[0].elapsed_time(ev[2]),
                         1e3 * (h1 - h0), 1e3 * (h2 - h0), 1e3 * (h3 - h2)))
    print(f"{a.workload}: step  from_csr  run+d2h  total | host: from_csr returns  total  free")
    for i, r in enumerate(rows):
        print(f"  {i:2d}  {r[0]:8.2f} {r[1]:8.2f} {r[2]:8.2f} | {r[3]:8.2f} {r[4]:8.2f} {r[5]:8.2f}")
    tot = sorted(r[2] for r in rows)
    print(f"  mean {sum(tot) / len(tot):.2f}  median {tot[len(tot) // 2]:.2f}  min {tot[0]:.2f}  max {tot[-1]:.2f}")
    # the same pinned columns copied by torch into a torch buffer (one stream, 128 MB chunks)
    d = torch.empty(t_col.numel(), dtype=torch.int32, device="cuda")
    CH = 1 << 25
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for b in range(0, t_col.numel(), CH):
            d[b:b + CH].copy_(t_col[b:b + CH], non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"  torch copy of the columns: {ms:.2f} ms, {t_col.numel() * 4 / ms / 1e6:.1f} GB/s")
    sys.stdout.flush()
    os._exit(0)  # pinned tensors were used on the library's stream: exit with them alive


if __name__ == "__main__":
    main()
