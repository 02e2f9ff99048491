"""Slab decomposition of a lowered stencil gradient over the GPUs of a node.

C5 (heat_3d 512^3, BASELINE.json configs[4]) is decomposed along the
outermost dimension: rank r owns a contiguous range of planes and keeps a
two-plane halo on each side. The single-device launch list (lowering.py,
after star-pair fusion and ping-pong placement) is rewritten per rank:

* each fused timestep (StarPairOp) becomes one grouped halo exchange of its
  source (width 2: X is recomputed on a one-plane halo from Y) and of the old
  intermediate (width 1), followed by the same kernel restricted to the
  owned planes, with masks/regions still in global coordinates;
* a reduction over a decomposed array becomes a local reduction over the
  owned planes plus an all-reduce of the scalar (the reference's dependent
  is a scalar sum, interpreter.py:447-451);
* broadcasts / whole-array fills run on the local slab (halo included).

The exchange is the only data-path communication: one send/recv pair per
neighbour per array per timestep, NCCL point-to-point over NVLink through
torch.distributed (gloo on CPU for the multi-process tests). Anything else
in the launch list is rejected loudly (UnsupportedConstruct).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import UnsupportedConstruct
from .lowering import BroadcastOp, Buffer, FillOp, Lowering, Op, ReduceOp, StarPairOp, whole_box

HALO = 2


@dataclass
class SlabPlan:
    N: int
    world: int
    rank: int
    halo: int = HALO

    def __post_init__(self):
        base, rem = divmod(self.N, self.world)
        self.own_lo = self.rank * base + min(self.rank, rem)
        self.own_hi = self.own_lo + base + (1 if self.rank < rem else 0)
        if self.own_hi - self.own_lo < self.halo:
            raise UnsupportedConstruct(f"slab of {self.own_hi - self.own_lo} planes is thinner than the halo")
        self.loc_lo = max(0, self.own_lo - self.halo)
        self.loc_hi = min(self.N, self.own_hi + self.halo)
        self.planes = self.loc_hi - self.loc_lo
        self.own_local = (self.own_lo - self.loc_lo, self.own_hi - self.loc_lo)

    def local_slice(self, arr):
        return arr[self.loc_lo:self.loc_hi]


class TorchComm:
    """Neighbour exchange and scalar all-reduce through torch.distributed."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist

    def plan_exchange(self, pairs):
        """Build the point-to-point op list for [(peer, send, recv)] once (the
        views are fixed for the executable's lifetime; rebuilding it every
        timestep is host time the GPU waits for at 8 ranks)."""
        dist = self.dist
        ops = []
        for peer, snd, rcv in pairs:
            ops.append(dist.P2POp(dist.isend, snd, peer))
            ops.append(dist.P2POp(dist.irecv, rcv, peer))
        return ops

    def run_exchange(self, ops):
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def exchange(self, pairs):
        """pairs: [(peer, send_tensor, recv_tensor)] posted together."""
        self.run_exchange(self.plan_exchange(pairs))

    def allreduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)


class HaloOp(Op):
    """Refresh the halo planes of decomposed buffers from the neighbours:
    [(buffer, width)], all exchanged in one grouped send/recv batch (one
    round trip per timestep instead of one per array)."""

    family = "halo"

    def __init__(self, items, plan: SlabPlan, comm):
        self.items, self.plan, self.comm = list(items), plan, comm
        self.reads = tuple(b for b, _ in self.items)
        self.writes = tuple(b for b, _ in self.items)

    def pairs(self, view):
        p = self.plan
        ol, oh = p.own_local
        pairs = []
        for buf, w in self.items:
            v = view(buf)
            if p.rank > 0:
                pairs.append((p.rank - 1, v[ol:ol + w], v[ol - w:ol]))
            if p.rank < p.world - 1:
                pairs.append((p.rank + 1, v[oh - w:oh], v[oh:oh + w]))
        return pairs

    def prepare(self, rt):
        # contiguous plane ranges of contiguous buffers: the views are the
        # buffers' own memory, fixed once they are placed
        plan, view = getattr(self.comm, "plan_exchange", None), getattr(rt, "view", None)
        self._ops = plan(self.pairs(view)) if plan is not None and view is not None else None

    def run(self, view):
        self.comm.exchange(self.pairs(view))

    def launch(self, rt, stream):
        ops = getattr(self, "_ops", None)
        if ops is not None:
            self.comm.run_exchange(ops)
        else:
            self.run(rt.view)

    def algorithmic_bytes(self) -> int:
        return sum(2 * w * (b.numel // b.shape[0]) * b.itemsize for b, w in self.items)


class AllReduceOp(Op):
    family = "allreduce"

    def __init__(self, buf: Buffer, comm):
        self.buf, self.comm = buf, comm
        self.reads = (buf,)
        self.writes = (buf,)

    def run(self, view):
        self.comm.allreduce_sum(view(self.buf).reshape(1))

    def launch(self, rt, stream):
        self.run(rt.view)


@dataclass
class DistLowered:
    low: Lowering
    inputs: dict
    outputs: dict
    seed_buf: object
    plan: SlabPlan


def decompose(lw, plan: SlabPlan, comm) -> DistLowered:
    """Rewrite a single-device Lowered gradient (api.lower_gradient) into the
    launch list of one rank."""
    ops = lw.low.ops
    pairs = [op for op in ops if isinstance(op, StarPairOp)]
    if not pairs:
        raise UnsupportedConstruct("slab decomposition needs a fused stencil program")
    shape = pairs[0].Z.shape
    if len(shape) != 3 or shape[0] != plan.N:
        raise UnsupportedConstruct("slab decomposition handles rank-3 stencil arrays split along dim 0")
    low = Lowering()
    local = {}
    lshape = (plan.planes,) + tuple(shape[1:])
    plane_elems = int(np.prod(shape[1:]))

    def loc(b: Buffer | None):
        if b is None:
            return None
        r = b.root()
        got = local.get(r.bid)
        if got is None:
            if r.shape == shape:
                got = low.new_buffer(r.name, lshape, r.kind, fresh=False)
            elif r.shape == ():
                got = low.new_buffer(r.name, (), r.kind, fresh=False)
            else:
                raise UnsupportedConstruct(f"slab decomposition: array '{r.name}' {r.shape} is not a slab array")
            local[r.bid] = got
        return got

    def own_view(b: Buffer) -> Buffer:
        v = low.new_buffer(b.name + "[own]", (plan.own_hi - plan.own_lo,) + tuple(shape[1:]), b.kind, fresh=False)
        v.alias_of = b
        v.offset = plan.own_local[0] * plane_elems
        return v

    for op in ops:
        if isinstance(op, StarPairOp):
            items = [(loc(op.Y), 2)]
            if op.X.root() is not op.Y.root():
                items.append((loc(op.X), 1))
            low.emit(HaloOp(items, plan, comm))
            new = StarPairOp(op.a, op.b, op.fa, op.fb, op.xwrite, op.dead)
            new.X, new.Y, new.Z = loc(op.X), loc(op.Y), loc(op.Z)
            new.xout, new.zout = loc(op.xout), loc(op.zout)
            new.plane0, new.zrange, new.global_d0 = plan.loc_lo, plan.own_local, plan.N
            new._refresh()
            low.emit(new)
        elif isinstance(op, ReduceOp) and op.x.root().shape == shape:
            if op.accumulate:
                raise UnsupportedConstruct("slab decomposition: accumulating reduction")
            low.emit(ReduceOp(own_view(loc(op.x)), loc(op.out), False))
            low.emit(AllReduceOp(loc(op.out), comm))
        elif isinstance(op, BroadcastOp):
            low.emit(BroadcastOp(loc(op.src), op.scale, loc(op.out), op.accumulate))
        elif isinstance(op, FillOp) and op.box == whole_box(op.dst.shape):
            low.emit(FillOp(loc(op.dst), whole_box(loc(op.dst).shape), op.value))
        else:
            raise UnsupportedConstruct(f"slab decomposition does not handle '{op.family}' launches")
    inputs = {k: loc(b) for k, b in lw.inputs.items()}
    outputs = {k: loc(b) for k, b in lw.outputs.items()}
    seed = loc(lw.seed_buf) if lw.seed_buf is not None else None
    return DistLowered(low, inputs, outputs, seed, plan)


def torch_empty_pinned(t):
    import torch

    return torch.empty(t.shape, dtype=t.dtype, pin_memory=True)


class SlabEngine:
    """One rank of a slab-decomposed gradient (bench.py under torchrun)."""

    def __init__(self, name: str, params: dict, rank: int, world: int, device):
        from . import workloads as W
        from .api import lower_gradient
        from .runtime import Executable

        self.name, self.params = name, dict(params)
        prog, bundle = W.load(name)
        self.program = prog
        shapes = W.input_shapes(prog, params)
        lw = lower_gradient(prog, bundle, params, shapes, fuse_small=True)
        N = next(iter(shapes.values()))[0]
        self.plan = SlabPlan(N, world, rank)
        self.dl = decompose(lw, self.plan, TorchComm())
        self.exe = Executable(self.dl.low, self.dl.inputs, self.dl.outputs, seed_buf=self.dl.seed_buf,
                              device=device, use_graph=False)
        self.device = device

    def local_inputs(self, seed=0) -> dict:
        import torch

        from . import workloads as W

        full = W.make_inputs(self.name, self.program, self.params, seed)
        return {k: torch.from_numpy(np.ascontiguousarray(self.plan.local_slice(v))).to(self.device)
                for k, v in full.items()}

    def step(self, inputs, seed=1.0, sync=False):
        self.exe.run(inputs, seed, sync=sync)

    def check(self):
        self.exe.check()

    def gradients(self, batches, seed=1.0):
        """Pipelined end-to-end calls on this rank (``Executable.run_pipelined``):
        value and owned planes of every gradient per batch of local slabs."""
        from .api import GradientResult

        lo, hi = self.plan.own_local
        outs = {"value": self.exe.output("value")}
        for key in self.exe.outputs:
            if key.startswith("grad:"):
                outs[key] = self.exe.output(key)[lo:hi]
        for host in self.exe.run_pipelined(batches, outs, seed):
            yield GradientResult(value=host.pop("value").numpy(),
                                 grads={k[5:]: v.numpy() for k, v in host.items()}, forward=None,
                                 backward=None, bundle=None)

    def gradient(self, host_local_inputs: dict, seed=1.0):
        """End-to-end call on this rank: H2D of the local slabs, the run,
        D2H of the value and of the owned planes of every gradient."""
        from .api import GradientResult

        self.exe.run(host_local_inputs, seed)
        value = self.exe.output_host("value")
        lo, hi = self.plan.own_local
        grads = {}
        for key in self.exe.outputs:
            if key.startswith("grad:"):
                t = self.exe.output(key)[lo:hi]
                h = torch_empty_pinned(t)
                h.copy_(t, non_blocking=True)
                grads[key[5:]] = h
        import torch

        torch.cuda.current_stream(self.device).synchronize()
        return GradientResult(value=value, grads={k: v.numpy() for k, v in grads.items()}, forward=None,
                              backward=None, bundle=None)

    def own_grad(self, name: str):
        g = self.exe.output("grad:" + name)
        lo, hi = self.plan.own_local
        return g[lo:hi]
