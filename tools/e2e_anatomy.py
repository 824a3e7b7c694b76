"""Where the end-to-end time of a bench workload goes (one B200).

    python tools/e2e_anatomy.py [--workload c3_rmat24_plp]

Times (CUDA events on the library stream, after a warm-up) the H2D copy of
the pinned host CSR alone, cd_graph_from_csr (copy + validation + finalize),
the detector on the resulting graph, and the whole e2e step of bench.py."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1304_4453_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3_rmat24_plp", choices=sorted(bench.WORKLOADS))
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

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        best = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            best.append(e0.elapsed_time(e1))
        return min(best)

    d_col = torch.empty_like(t_col, device="cuda")
    with torch.cuda.stream(stream):
        ms_h2d = timed(lambda: d_col.copy_(t_col, non_blocking=True))
    nbytes = t_off.numel() * 8 + t_col.numel() * 4 + (t_w.numel() * 4 if t_w is not None else 0)
    del d_col
    hold = {}

    def build():
        hold["g"] = None
        hold["g"] = P.Graph.from_csr(n, t_off.numpy(), t_col.numpy(), None if t_w is None else t_w.numpy(), ctx=ctx)

    ms_build = timed(build)
    gg = hold["g"]
    ms_run = timed(lambda: bench.run_device(P, gg, wl["algo"], h_out, report=False))

    def e2e():
        build()
        bench.run_device(P, hold["g"], wl["algo"], h_out, report=False)

    ms_e2e = timed(e2e)
    print(f"{a.workload}: bytes {nbytes / 1e9:.3f} GB; col H2D alone {ms_h2d:.2f} ms "
          f"({t_col.numel() * 4 / ms_h2d / 1e6:.1f} GB/s); from_csr {ms_build:.2f} ms; run (host out) "
          f"{ms_run:.2f} ms; e2e {ms_e2e:.2f} ms")
    # exit here, with every local alive: the pinned tensors were used on the
    # library's stream (torch records an event there when they are freed), so
    # they must not outlive the context -- nor be freed after it at teardown
    sys.stdout.flush()
    os._exit(0)


if __name__ == "__main__":
    main()
    sys.stdout.flush()
    os._exit(0)  # skip interpreter teardown: pinned torch tensors outlive the library context
