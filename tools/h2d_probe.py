import time, torch, numpy as np, statistics
dev = torch.device("cuda", 0)
n = 104**3
src = np.random.default_rng(0).standard_normal(n)
dst = torch.empty(n, dtype=torch.float64, device=dev)
buf = torch.empty(n, dtype=torch.float64, pin_memory=True)
def t(f, reps=20):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    return round(statistics.median(ts), 3)
s = torch.from_numpy(src)
def single(): buf.copy_(s); dst.copy_(buf, non_blocking=True)
def chunks(k):
    def f():
        step = -(-n // k)
        for a in range(0, n, step):
            b = min(n, a + step); buf[a:b].copy_(s[a:b]); dst[a:b].copy_(buf[a:b], non_blocking=True)
    return f
def host_only(): buf.copy_(s)
def pageable(): dst.copy_(s)
def npcopy(): np.copyto(buf.numpy(), src); dst.copy_(buf, non_blocking=True)
print({"threads": torch.get_num_threads(), "host_only": t(host_only), "single": t(single), "chunks4": t(chunks(4)), "chunks8": t(chunks(8)), "chunks16": t(chunks(16)), "pageable": t(pageable), "npcopy": t(npcopy)})
