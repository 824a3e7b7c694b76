"""Host->device copy rate of 2.2 GB from pinned memory: one stream vs chunks
alternating over 2 / 4 streams (does a second copy engine add PCIe rate?)."""
import torch

N = 2217280600 // 4
src = torch.empty(N, dtype=torch.int32).pin_memory()
dst = torch.empty(N, dtype=torch.int32, device="cuda")
CH = 1 << 25
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    best = 1e9
    for rep in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in streams:
            s.wait_event(e0)
        for i, b in enumerate(range(0, N, CH)):
            s = streams[i % ns]
            with torch.cuda.stream(s):
                dst[b:b + CH].copy_(src[b:b + CH], non_blocking=True)
        for s in streams:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"streams {ns}: {best:.2f} ms, {N * 4 / best / 1e6:.1f} GB/s", flush=True)
