"""H2D of 9 MB from pinned memory: one stream vs split over 2 / 4 streams."""
import statistics, time, torch
dev = torch.device("cuda", 0)
n = 104 ** 3
buf = torch.randn(n, dtype=torch.float64).pin_memory()
dst = torch.empty(n, dtype=torch.float64, device=dev)
streams = [torch.cuda.Stream() for _ in range(4)]
def t(f, reps=30):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(statistics.median(ts), 3)
def split(k):
    def f():
        step = -(-n // k)
        for i, a in enumerate(range(0, n, step)):
            b = min(n, a + step)
            with torch.cuda.stream(streams[i]):
                dst[a:b].copy_(buf[a:b], non_blocking=True)
    return f
out = {"one": t(lambda: dst.copy_(buf, non_blocking=True)), "two": t(split(2)), "four": t(split(4))}
d2h = torch.empty(n, dtype=torch.float64).pin_memory()
out["d2h_one"] = t(lambda: d2h.copy_(dst, non_blocking=True))
print(out)
