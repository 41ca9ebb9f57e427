"""PCIe copy-rate probe for the e2e leg: pinned H2D / D2H alone, H2D split over 1/2/4 streams, and
H2D concurrent with D2H (CUDA events, median of 5)."""
import statistics

import torch

MB = 1 << 20
h = torch.empty(384 * MB, dtype=torch.uint8).pin_memory()
d = torch.empty(384 * MB, dtype=torch.uint8, device="cuda")
ho = torch.empty(256 * MB, dtype=torch.uint8).pin_memory()
do = torch.empty(256 * MB, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def timed(fn):
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts[1:])


def h2d(ns):
    def f():
        n = h.numel() // ns
        cur = torch.cuda.current_stream()
        for i, s in enumerate(streams[:ns]):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * n:(i + 1) * n].copy_(h[i * n:(i + 1) * n], non_blocking=True)
    return f


def both(ns):
    def f():
        cur = torch.cuda.current_stream()
        streams[3].wait_stream(cur)
        with torch.cuda.stream(streams[3]):
            ho.copy_(do, non_blocking=True)
        n = h.numel() // ns
        for i, s in enumerate(streams[:ns]):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * n:(i + 1) * n].copy_(h[i * n:(i + 1) * n], non_blocking=True)
    return f


for ns in (1, 2, 3):
    t = timed(h2d(ns))
    print(f"H2D 384 MB over {ns} stream(s): {t:.3f} ms = {384 * MB / t / 1e6:.1f} GB/s")
t = timed(lambda: ho.copy_(do, non_blocking=True))
print(f"D2H 256 MB: {t:.3f} ms = {256 * MB / t / 1e6:.1f} GB/s")
for ns in (1, 2):
    t = timed(both(ns))
    print(f"H2D 384 MB ({ns} streams) || D2H 256 MB: {t:.3f} ms")
