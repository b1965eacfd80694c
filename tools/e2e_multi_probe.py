import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2012_00866_b200 as h
import workloads as W
w = W.make("C2")
dev = torch.device("cuda", 0)
hu = torch.from_numpy(w.units).pin_memory(); ho = torch.from_numpy(w.offsets).pin_memory()
du = torch.empty(hu.shape, dtype=hu.dtype, device=dev); do = torch.empty(ho.shape, dtype=ho.dtype, device=dev)
comm = h.husky_comm_create(0, 1, h.husky_comm_unique_id()); h.multi._WORLD[comm.value] = 1
du.copy_(hu); do.copy_(ho)
for i in range(3): h.sort_multi(comm, 0, du, do, 0)
torch.cuda.synchronize()
def t(f, k=3):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts)
print("h2d", t(lambda: (du.copy_(hu, non_blocking=True), do.copy_(ho, non_blocking=True))))
print("sort_multi", t(lambda: h.sort_multi(comm, 0, du, do, 0)))
p, su, so, _ = h.sort_multi(comm, 0, du, do, 0)
hp = torch.empty(p.numel(), dtype=torch.int32).pin_memory(); hsu = torch.empty(su.numel(), dtype=su.dtype).pin_memory(); hso = torch.empty(so.numel(), dtype=torch.int64).pin_memory()
print("d2h", t(lambda: (hp.copy_(p, non_blocking=True), hsu.copy_(su, non_blocking=True), hso.copy_(so, non_blocking=True))))
print("sort_host", t(lambda: h.sort(0, du, do)))
# the bench loop, step by step
cap_n, cap_u = 2 * w.n + 1024, 2 * w.units.size + 1024
hp2 = torch.empty(cap_n, dtype=torch.int32).pin_memory(); hsu2 = torch.empty(cap_u, dtype=torch.uint8).pin_memory(); hso2 = torch.empty(cap_n + 1, dtype=torch.int64).pin_memory()
def step():
    du.copy_(hu, non_blocking=True); do.copy_(ho, non_blocking=True)
    p, su, so, _ = h.sort_multi(comm, 0, du, do, 0)
    hp2[:p.numel()].copy_(p, non_blocking=True); hsu2[:su.numel()].copy_(su, non_blocking=True); hso2[:so.numel()].copy_(so, non_blocking=True)
print("bench step", t(step))
def step2():
    du.copy_(hu, non_blocking=True); do.copy_(ho, non_blocking=True)
    torch.cuda.synchronize()
    p, su, so, _ = h.sort_multi(comm, 0, du, do, 0)
    torch.cuda.synchronize()
    hp2[:p.numel()].copy_(p, non_blocking=True); hsu2[:su.numel()].copy_(su, non_blocking=True); hso2[:so.numel()].copy_(so, non_blocking=True)
print("bench step with syncs", t(step2))
