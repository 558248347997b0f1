"""Device->host copy bandwidth on this box (pinned host memory): one stream vs two, chunk
sizes. Explains the e2e bound of bench.py (its outputs leave the GPU every step)."""
import time

import torch

n = 168 << 20  # one bench step's outputs (8 views x 20 B x 1024^2)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def bw(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return n * reps / (time.perf_counter() - t0) / 1e9


def chunks(k, streams):
    def f():
        step = n // k
        for i in range(k):
            with torch.cuda.stream(streams[i % len(streams)]):
                host[i * step:(i + 1) * step].copy_(dev[i * step:(i + 1) * step], non_blocking=True)
    return f


for k in (1, 8, 64):
    print(f"D2H {k:3d} chunks, 1 stream : {bw(chunks(k, [s1])):6.1f} GB/s")
    print(f"D2H {k:3d} chunks, 2 streams: {bw(chunks(k, [s1, s2])):6.1f} GB/s")
print(f"H2D 1 chunk              : {bw(lambda: dev.copy_(h2, non_blocking=True)):6.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        host.copy_(dev, non_blocking=True)
    with torch.cuda.stream(s2):
        dev.copy_(h2, non_blocking=True)


print(f"D2H + H2D concurrently   : {bw(both):6.1f} GB/s each")
