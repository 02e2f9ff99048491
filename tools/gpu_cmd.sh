python -m pytest tests/test_gpu_r2.py tests/test_gpu.py -q -x -k "seidel" > gpurun_out/r2_seidel.log 2>&1
python - >> gpurun_out/r2_seidel.log 2>&1 <<'PY'
import time, torch, numpy as np, os
from paper_2509_02197_b200 import Engine
from paper_2509_02197_b200.api import load_bundle
from paper_2509_02197_b200.ir import load_program
stem = "paper_2509_02197_b200/programs/corpus_seidel_stencil"
prog = load_program(stem + ".fwd.json"); b = load_bundle(stem + ".bwd.json", stem + ".fwdreq.json")
params = {"N": 400, "TSTEPS": 100}
eng = Engine(prog, b, params)
dev = {"A": torch.rand(400, 400, dtype=torch.float64, device="cuda")}
for _ in range(3): eng.step(dev)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5): eng.step(dev)
e.record(); torch.cuda.synchronize()
print("seidel N=400 T=100 ms per gradient", s.elapsed_time(e) / 5)
PY
