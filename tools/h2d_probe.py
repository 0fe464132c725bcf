"""Host->device bandwidth from pinned memory with 1..4 concurrent streams."""
import torch
N = 8 * 25_600_000
h = torch.empty(N, dtype=torch.float32).pin_memory()
h.fill_(1.0)
d = torch.empty(N, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    parts = torch.chunk(torch.arange(N), ns)
    best = 1e9
    for rep in range(5):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        cur = torch.cuda.current_stream()
        for s, p in zip(streams, torch.chunk(torch.arange(N), ns)):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                lo, hi = int(p[0]), int(p[-1]) + 1
                d[lo:hi].copy_(h[lo:hi], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{ns} streams: {N*4/best/1e6:.1f} GB/s ({best:.2f} ms)")
