"""Do D2H / H2D copies on side streams overlap a compute kernel stream on this box?"""
import time, torch
dev = torch.device("cuda", 0)
n = 33554432
a = torch.randn(8192, 8192, device=dev)
hout = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(8)]
dout = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(8)]
cs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
def compute():
    with torch.cuda.stream(cs):
        for _ in range(20): torch.mm(a, a)
def d2h():
    with torch.cuda.stream(ds):
        for x, y in zip(hout, dout): x.copy_(y, non_blocking=True)
for name, fns in [("compute", [compute]), ("d2h", [d2h]), ("both", [compute, d2h])]:
    for f in fns: f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        for f in fns: f()
    torch.cuda.synchronize()
    print(name, round((time.perf_counter() - t) / 3 * 1e3, 1), "ms")
