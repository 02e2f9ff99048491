"""Host-side enqueue cost of one eager step of the C5 launch list: the
single-device list and a two-rank slab list (rank 0, exchange calls stubbed:
NCCL's own host cost is not included). Reports host ms per step next to the
device ms per step, to tell whether an eager multi-rank step is host-bound."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_02197_b200 import workloads as W  # noqa: E402
from paper_2509_02197_b200.api import lower_gradient  # noqa: E402
from paper_2509_02197_b200.decomp import SlabPlan, decompose  # noqa: E402
from paper_2509_02197_b200.runtime import Executable  # noqa: E402


class NullComm:
    def plan_exchange(self, pairs):
        return [0]

    def run_exchange(self, ops):
        pass

    def exchange(self, pairs):
        pass

    def allreduce_sum(self, t):
        pass


def measure(exe, inputs, reps=3):
    exe.run(inputs, sync=True)
    best_host, best_dev = 1e9, 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        exe.launch_all()
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        best_host = min(best_host, (t1 - t0) * 1e3)
        best_dev = min(best_dev, e0.elapsed_time(e1))
    return best_host, best_dev


name, params = W.CONFIGS["C5/heat_3d"]
prog, b = W.load(name)
shapes = W.input_shapes(prog, params)
full = W.make_inputs(name, prog, params, 0)
lw = lower_gradient(prog, b, params, shapes, fuse_small=True)
exe = Executable(lw.low, lw.inputs, lw.outputs, seed_buf=lw.seed_buf, use_graph=False)
dev = {k: torch.from_numpy(v).cuda() for k, v in full.items()}
h, d = measure(exe, dev)
print(f"single device, eager: {len(exe.ops)} ops, host {h:.2f} ms, device {d:.2f} ms per step")
del exe
for world in (2, 4, 8):
    lw = lower_gradient(prog, b, params, shapes, fuse_small=True)
    plan = SlabPlan(params["N"], world, 0)
    dl = decompose(lw, plan, NullComm())
    exe = Executable(dl.low, dl.inputs, dl.outputs, seed_buf=dl.seed_buf, use_graph=False)
    exe.comm_stream = torch.cuda.Stream()
    loc = {k: torch.from_numpy(plan.local_slice(v).copy()).cuda() for k, v in full.items()}
    h, d = measure(exe, loc)
    print(f"slab rank 0 of {world}, eager, exchanges stubbed: {len(exe.ops)} ops, host {h:.2f} ms, "
          f"device {d:.2f} ms per step")
    del exe

# per-launch device times of one timestep of the 8-rank list (eager, events)
lw = lower_gradient(prog, b, params, shapes, fuse_small=True)
plan = SlabPlan(params["N"], 8, 3)
dl = decompose(lw, plan, NullComm())
exe = Executable(dl.low, dl.inputs, dl.outputs, seed_buf=dl.seed_buf, use_graph=False)
exe.comm_stream = torch.cuda.Stream()
loc = {k: torch.from_numpy(plan.local_slice(v).copy()).cuda() for k, v in full.items()}
exe.run(loc, sync=True)
rows = exe.timed_eager(loc)
tot = {}
for fam, op, ms in rows:
    key = fam
    if isinstance(getattr(op, "edges", None), list):
        key = f"edges ({len(op.edges)} ranges)"
    elif fam == "star_pair":
        lo, hi = op.zrange
        key = f"star_pair[{hi - lo} planes]"
    tot.setdefault(key, [0, 0.0])
    tot[key][0] += 1
    tot[key][1] += ms
for k, (n, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"  rank 3 of 8: {k:24s} {n:4d} launches {ms:8.2f} ms  {ms / n * 1e3:7.1f} us each")
