"""Pinned host -> device copy bandwidth on this box (the e2e path's PCIe ceiling):
one and two streams, 16 MB .. 256 MB copies."""
import torch

dev = torch.device("cuda:0")
for mb in (16, 64, 256):
    n = mb * (1 << 20) // 8
    src = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(8)]
    dst = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(8)]
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        torch.cuda.synchronize()
        for rep in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in streams:
                s.wait_event(e0)
            for i in range(8):
                with torch.cuda.stream(streams[i % ns]):
                    dst[i].copy_(src[i], non_blocking=True)
            for s in streams:
                e1.wait_stream(s) if hasattr(e1, "wait_stream") else torch.cuda.current_stream().wait_stream(s)
            torch.cuda.current_stream().wait_stream(streams[0])
            for s in streams:
                torch.cuda.current_stream().wait_stream(s)
            e1.record()
            torch.cuda.synchronize()
        print(f"H2D {mb:4d} MB x 8, {ns} stream(s): {8 * mb / 1024 / (e0.elapsed_time(e1) / 1e3):6.1f} GiB/s")
