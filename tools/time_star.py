"""Per-launch time of the fused star-pair kernel on heat_3d 512^3 (a few
timesteps, graph replay) for the library in GFB_LIBRARY; parity-checked
against the default build's result at N=66 first."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_02197_b200 import Engine, workloads as W  # noqa: E402

name = "heat_3d"
prog, b = W.load(name)
# parity at a small size against the oracle
from oracle import interp as O  # noqa: E402

params = {"N": 66, "TSTEPS": 4}
inp = W.make_inputs(name, prog, params, 0)
v, g, _ = O.gradient(prog, b.backward, b.forwarding, b.required, inp, params)
eng = Engine(prog, b, params)
res = eng.gradient(inp)
err = float(np.max(np.abs(res.grads["A"] - g["A"]) / np.maximum(1, np.abs(g["A"]))))
params = {"N": 512, "TSTEPS": 6}
eng = Engine(prog, b, params)
dev = {k: torch.from_numpy(v).cuda() for k, v in W.make_inputs(name, prog, params, 0).items()}
for _ in range(3):
    eng.step(dev)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    eng.step(dev)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
n = sum(1 for op in eng.exe.ops if op.family == "star_pair")
print(f"{os.environ.get('GFB_LIBRARY', 'default')}: grad err {err:.1e}, {ms / n:.4f} ms per fused launch ({n} launches)")
