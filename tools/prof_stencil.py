"""Small driver for ncu captures of the stencil sweeps: heat_3d N=512 with a
few timesteps, one eager gradient (forward + adjoint sweeps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_02197_b200 import Engine, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "heat_3d"
params = {"N": int(sys.argv[2]) if len(sys.argv) > 2 else 512, "TSTEPS": int(sys.argv[3]) if len(sys.argv) > 3 else 3}
prog, b = W.load(name)
os.environ["GFB_GRAPH"] = "0"
eng = Engine(prog, b, params)
inp = {k: torch.from_numpy(v).cuda() for k, v in W.make_inputs(name, prog, params, 0).items()}
eng.step(inp)
torch.cuda.synchronize()
print("ok", float(eng.exe.output("value")))
