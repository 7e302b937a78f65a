"""Copy-engine interference probe: while a 4.29 GB pinned H2D reload runs on
one stream, how long does a tiny H2D (a step's input descriptors) on another
stream wait?  Variants: the reload as one copy, as per-layer chunks (64 x 67 MB),
as 16 MB chunks; the tiny copy as H2D and as D2H."""
import time

import torch

N = 4 * 1024**3 + 200 * 1024**2
host = torch.empty(N, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
small_h = torch.zeros(4096, dtype=torch.uint8, pin_memory=True)
small_d = torch.zeros(4096, dtype=torch.uint8, device="cuda")
a, b = torch.cuda.Stream(), torch.cuda.Stream()


def run(chunks, direction):
    torch.cuda.synchronize()
    step = N // chunks
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(a):
        for i in range(chunks):
            dev[i * step:(i + 1) * step].copy_(host[i * step:(i + 1) * step], non_blocking=True)
    time.sleep(0.005)  # the reload is under way
    with torch.cuda.stream(b):
        e0.record()
        for _ in range(3):
            if direction == "h2d":
                small_d.copy_(small_h, non_blocking=True)
            else:
                small_h.copy_(small_d, non_blocking=True)
        e1.record()
    e1.synchronize()
    t_small = e0.elapsed_time(e1)
    torch.cuda.synchronize()
    return t_small


for direction in ("h2d", "d2h"):
    for chunks in (1, 64, 256):
        ts = [run(chunks, direction) for _ in range(3)]
        print(f"small {direction} while a 4.3 GB H2D in {chunks} chunks runs: {[round(t, 2) for t in ts]} ms", flush=True)
