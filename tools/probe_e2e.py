"""Break the end-to-end heat_3d 512^3 call into its parts (H2D, device
gradient, D2H, result assembly) to see where e2e time goes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_02197_b200 import Engine, workloads as W  # noqa: E402

name, params = W.CONFIGS["C5/heat_3d"]
prog, b = W.load(name)
eng = Engine(prog, b, params)
host = {k: torch.from_numpy(v).pin_memory() for k, v in W.make_inputs(name, prog, params, 0).items()}
dev = {k: v.cuda() for k, v in host.items()}
for _ in range(2):
    eng.step(dev)
torch.cuda.synchronize()


def t(f, n=3):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1000


print("h2d 2 inputs (pinned)   %.1f ms" % t(lambda: eng.exe.load_inputs(host)))
print("device step             %.1f ms" % t(lambda: eng.step(dev)))
print("output_host grad        %.1f ms" % t(lambda: eng.exe.output_host("grad:A")))
g = eng.exe.output("grad:A")
hb = torch.empty(g.shape, dtype=g.dtype, pin_memory=True)
print("d2h into kept pinned    %.1f ms" % t(lambda: hb.copy_(g, non_blocking=True)))
print("pinned alloc 1 GiB      %.1f ms" % t(lambda: torch.empty(g.shape, dtype=g.dtype, pin_memory=True)))
print("np copy of 1 GiB        %.1f ms" % t(lambda: hb.numpy().copy()))
print("full gradient()         %.1f ms" % t(lambda: eng.gradient(host)))
