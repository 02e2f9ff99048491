python -m pytest tests/test_gpu.py -q -x -k "conv2d or contract or c4_full or golden" > gpurun_out/r2_conv_tests.log 2>&1
python tools/bench_all.py --no-cpu --steps 20 --only C4/conv2d_bias > gpurun_out/r2_conv.jsonl 2> gpurun_out/r2_conv.err
GFB_CONTRACT_TC=0 python tools/bench_all.py --no-cpu --steps 20 --only C4/conv2d_bias >> gpurun_out/r2_conv.jsonl 2>> gpurun_out/r2_conv.err
python - >> gpurun_out/r2_conv.jsonl 2>&1 <<'PY'
import torch, numpy as np, json
from paper_2509_02197_b200 import Engine, workloads as W
name, params = W.CONFIGS['C4/conv2d_bias']
prog, b = W.load(name)
eng = Engine(prog, b, params)
dev = {k: torch.from_numpy(v).cuda() for k, v in W.make_inputs(name, prog, params, 0).items()}
eng.step(dev); torch.cuda.synchronize()
rows = eng.exe.timed_eager(dev)
for fam, op, ms in rows:
    print(fam, round(ms * 1e3, 1), "us", type(op).__name__, getattr(op, "M", ""), getattr(op, "N", ""), getattr(op, "K", ""))
PY
