"""Developer probe: pinned host <-> device copy rates for cfg5-sized state
vectors (102 MB), one direction at a time and both directions at once."""
import json
import time

import torch

n = 3 * 8489664
h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(3)]
d = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(3)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


out = {}
out["h2d_ms"] = timed(lambda: d[0].copy_(h[0], non_blocking=True))
out["d2h_ms"] = timed(lambda: h[1].copy_(d[1], non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(s2):
        h[1].copy_(d[1], non_blocking=True)


out["h2d_and_d2h_ms"] = timed(both)


def two_h2d():
    with torch.cuda.stream(s1):
        d[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(s2):
        d[1].copy_(h[1], non_blocking=True)


out["two_h2d_ms"] = timed(two_h2d)
out["bytes"] = n * 4
print(json.dumps(out))
