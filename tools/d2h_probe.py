"""Pinned D2H bandwidth: one 1.68 GB copy, 16 chunks on one stream, and 16
chunks over two streams (copy-engine concurrency)."""
import torch

N = 1_679_478_544
d = torch.empty(N, dtype=torch.uint8, device="cuda")
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d.fill_(1)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return N / (best / 1e3) / 1e9


def one():
    h.copy_(d, non_blocking=True)


def chunks(nst):
    c = N // 16
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    for i in range(16):
        st = s1 if (nst == 1 or i % 2 == 0) else s2
        with torch.cuda.stream(st):
            h[i * c:(i + 1) * c].copy_(d[i * c:(i + 1) * c], non_blocking=True)


print("single copy   GB/s %.1f" % t(one))
print("16 chunks x1  GB/s %.1f" % t(lambda: chunks(1)))
print("16 chunks x2  GB/s %.1f" % t(lambda: chunks(2)))
