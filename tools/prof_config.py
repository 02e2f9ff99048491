"""ncu driver: one eager gradient step of a BASELINE config (per-launch
kernels visible), e.g. python tools/prof_config.py C4/softmax"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GFB_GRAPH"] = "0"
import torch  # noqa: E402

from paper_2509_02197_b200 import Engine, workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4/softmax"
name, params = W.CONFIGS[cfg]
prog, b = W.load(name)
eng = Engine(prog, b, params)
inp = {k: torch.from_numpy(v).cuda() for k, v in W.make_inputs(name, prog, params, 0).items()}
eng.step(inp)
eng.step(inp)
torch.cuda.synchronize()
print("ok", float(eng.exe.output("value")))
