"""HBM direction probe: write-only (fill), read-only (sum / custom read), copy, CUDA events, best of 10."""
import torch

N = 8 << 30  # bytes
a = torch.empty(N // 4, dtype=torch.int32, device="cuda")
b = torch.empty(N // 4, dtype=torch.int32, device="cuda")
a.fill_(1)
torch.cuda.synchronize()


def best(fn, nbytes, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    t = min(out)
    return nbytes / (t / 1e3) / 1e9


print("write-only fill_   GB/s %.0f" % best(lambda: b.fill_(7), N))
print("write-only zero_   GB/s %.0f" % best(lambda: b.zero_(), N))
print("read-only  sum     GB/s %.0f" % best(lambda: a.sum(dtype=torch.int64), N))
print("copy (r+w) copy_   GB/s %.0f" % best(lambda: b.copy_(a), 2 * N))
