import torch, time
dev = torch.device("cuda", 0)
n = 33554432
hin = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(11)]
din = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(11)]
hout = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(8)]
dout = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(8)]
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
def h2d(s):
    with torch.cuda.stream(s):
        for a, b in zip(din, hin): a.copy_(b, non_blocking=True)
def d2h(s):
    with torch.cuda.stream(s):
        for a, b in zip(hout, dout): a.copy_(b, non_blocking=True)
for name, fn in [("h2d", lambda: h2d(s1)), ("d2h", lambda: d2h(s2)), ("both", lambda: (h2d(s1), d2h(s2)))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(name, round(dt * 1e3, 1), "ms")
