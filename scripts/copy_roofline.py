"""Dev: practical HBM roofline for the bench transfer sizes -- torch copy /
add kernels over the same byte counts, L2 flushed, CUDA events."""
import torch

torch.cuda.set_device(0)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(64 << 20, device="cuda")
sink = torch.empty((), device="cuda")


def t(fn, nbytes, label):
    ts = []
    for it in range(12):
        with torch.cuda.stream(s):
            flush.zero_()
            torch.sum(rd, 0, out=sink)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    med = ts[len(ts) // 2]
    print("%-34s %8.1f us  %7.0f GB/s" % (label, med, nbytes / med / 1e3), flush=True)


for mb in (50, 67, 134, 512):
    n = mb * (1 << 20) // 4
    x = torch.randn(n, device="cuda")
    y = torch.empty_like(x)
    t(lambda: y.copy_(x), 2 * n * 4, "copy %d MB -> %d MB" % (mb, mb))
for mb in (67, 134):
    n = mb * (1 << 20) // 4
    a, b, c = torch.randn(n, device="cuda"), torch.randn(n, device="cuda"), torch.empty(n, device="cuda")
    t(lambda: torch.add(a, b, out=c), 3 * n * 4, "add 2x%d MB -> %d MB" % (mb, mb))
n = 134 * (1 << 20) // 4
x = torch.randn(n, device="cuda")
t(lambda: x.sum(), n * 4, "sum 134 MB")
