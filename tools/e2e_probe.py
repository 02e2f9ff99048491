"""Where does the end-to-end C5 step go? Times H2D / D2H alone and the
pipelined Engine.gradients per-step wall intervals (diagnostic, not a bench)."""
import time

import torch

from paper_2509_02197_b200 import Engine, workloads as W

name, params = W.CONFIGS["C5/heat_3d"]
prog, b = W.load(name)
eng = Engine(prog, b, params)
host_np = W.make_inputs(name, prog, params, 0)
host = {k: torch.from_numpy(v).pin_memory() for k, v in host_np.items()}
dev = {k: v.cuda() for k, v in host.items()}
for _ in range(3):
    eng.step(dev)
torch.cuda.synchronize()


def t(fn, n=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


d = torch.empty_like(dev["A"])
h = torch.empty(d.shape, dtype=d.dtype, pin_memory=True)
print("H2D 1 GiB ms", t(lambda: d.copy_(host["A"], non_blocking=True)))
print("D2H 1 GiB ms", t(lambda: h.copy_(d, non_blocking=True)))
print("step ms", t(lambda: eng.step(dev)))
t0 = time.perf_counter()
torch.empty(d.shape, dtype=d.dtype, pin_memory=True)
print("fresh pinned alloc ms", (time.perf_counter() - t0) * 1e3)
for n in (8, 16):
    for _ in eng.gradients([host] * 3):
        pass
    stamps = []
    t0 = time.perf_counter()
    for r in eng.gradients([host] * n):
        stamps.append(time.perf_counter() - t0)
    print(n, "pipelined total ms", stamps[-1] * 1e3, "per-step intervals", [round((b - a) * 1e3, 1) for a, b in zip([0] + stamps, stamps)])
