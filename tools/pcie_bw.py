"""Host<->device copy bandwidth (pinned and pageable) for the e2e roofline."""
import time

import torch

n = 256 * 1024 * 1024  # bytes
dev = torch.device("cuda", 0)
d = torch.empty(n, dtype=torch.uint8, device=dev)
d2 = torch.empty(n, dtype=torch.uint8, device=dev)
hp = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hp2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hq = torch.empty(n, dtype=torch.uint8)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


print("H2D pinned  GB/s", n / t(lambda: d.copy_(hp, non_blocking=True)) / 1e9)
print("D2H pinned  GB/s", n / t(lambda: hp.copy_(d, non_blocking=True)) / 1e9)
print("H2D pageable GB/s", n / t(lambda: d.copy_(hq)) / 1e9)
print("D2H pageable GB/s", n / t(lambda: hq.copy_(d)) / 1e9)


def both():
    with torch.cuda.stream(s1):
        d.copy_(hp, non_blocking=True)
    with torch.cuda.stream(s2):
        hp2.copy_(d2, non_blocking=True)


print("H2D+D2H concurrent GB/s each", n / t(both) / 1e9)
