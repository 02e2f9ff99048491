"""Slab decomposition of a lowered stencil gradient over the GPUs of a node.

C5 (heat_3d 512^3, BASELINE.json configs[4]) is decomposed along the
outermost dimension: rank r owns a contiguous range of planes and keeps a
two-plane halo on each side. The single-device launch list (lowering.py,
after star-pair fusion and ping-pong placement) is rewritten per rank:

* each fused timestep (StarPairOp) becomes
    - one grouped halo exchange (HaloOp) of its source (width 2: X is
      recomputed on a one-plane halo from Y) and of the old intermediate
      (width 1), issued on a communication stream once the previous
      timestep's edge planes are written;
    - the same kernel on the interior planes [own_lo + 2, own_hi - 2), which
      read no halo plane and run on the compute stream WHILE the exchange
      is in flight;
    - the kernel on the two edge plane ranges (two planes at each slab end)
      on the communication stream right behind the exchange, so a
      timestep's edges run beside its interior (EdgeOp; StreamMark /
      StreamJoin carry the cross-stream order: the interior of timestep
      t + 1 waits for the edges of t, the edges of t wait for the interior
      of t - 1, whose planes they read);
  masks / regions stay in global coordinates (plane0 in the descriptor);
* a reduction over a decomposed array becomes a local reduction over the
  owned planes plus an all-reduce of the scalar (the reference's dependent
  is a scalar sum, interpreter.py:447-451);
* broadcasts / whole-array fills run on the local slab (halo included).

The exchange is the only data-path communication: one send/recv pair per
neighbour per array per timestep, NCCL point-to-point over NVLink through
torch.distributed (gloo on CPU for the multi-process tests). With a single
rank there is nothing to exchange: the rewritten list has no communication
op and is captured in a CUDA graph like the single-device engine. Anything
else in the launch list is rejected loudly (UnsupportedConstruct).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import UnsupportedConstruct
from .lowering import BroadcastOp, Buffer, FillOp, Lowering, Op, ReduceOp, StarPairOp, whole_box

HALO = 2
SLAB_INTERIOR_TPM = 24  # planes per CTA of a slab's interior launch (see decompose)


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
    """Neighbour exchange and scalar all-reduce through torch.distributed
    (NCCL on the GPUs of a node; gloo in the CPU tests). ``group`` is an
    optional process group; peers are ranks within it."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def plan_exchange(self, pairs):
        """Build the point-to-point op list for [(peer, send, recv)] once (the
        views are fixed for the executable's lifetime; rebuilding it every
        timestep is host time the GPU waits for at 8 ranks)."""
        dist = self.dist
        ops = []
        for peer, snd, rcv in pairs:
            ops.append(dist.P2POp(dist.isend, snd, self._peer(peer), self.group))
            ops.append(dist.P2POp(dist.irecv, rcv, self._peer(peer), self.group))
        return ops

    def run_exchange(self, ops):
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def exchange(self, pairs):
        """pairs: [(peer, send_tensor, recv_tensor)] posted together."""
        self.run_exchange(self.plan_exchange(pairs))

    def allreduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)


class HaloOp(Op):
    """Refresh the halo planes of decomposed buffers from the neighbours:
    [(buffer, width)], all exchanged in one grouped send/recv batch (one
    round trip per timestep instead of one per array)."""

    family = "halo"

    def __init__(self, items, plan: SlabPlan, comm, first=False):
        self.items, self.plan, self.comm = list(items), plan, comm
        self.first = first  # first timestep of a chain: join the compute stream
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
        comm_stream = getattr(rt, "comm_stream", None)
        if ops is None:
            self.run(rt.view)
            return
        if comm_stream is None:
            self.comm.run_exchange(ops)
            return
        import torch

        # the exchange sends the edge planes of the previous timestep, which
        # ran on this stream; the first timestep of a chain starts from what
        # the compute stream produced (inputs, seeds, broadcasts)
        if self.first:
            comm_stream.wait_stream(torch.cuda.current_stream(rt.device))
            rt._ev_int = rt._ev_int_prev = rt._ev_edges = None
        with torch.cuda.stream(comm_stream):
            self.comm.run_exchange(ops)

    def algorithmic_bytes(self) -> int:
        """Bytes the exchange moves out of this rank (both neighbours)."""
        nb = (self.plan.rank > 0) + (self.plan.rank < self.plan.world - 1)
        return sum(nb * w * (b.numel // b.shape[0]) * b.itemsize for b, w in self.items)


class StreamMark(Op):
    """After a timestep's interior on the compute stream: record it (the
    next timestep's edges read its planes)."""

    family = "halo_wait"

    def __init__(self):
        self.reads = self.writes = ()

    def launch(self, rt, stream):
        if getattr(rt, "comm_stream", None) is None:
            return
        import torch

        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(rt.device))
        rt._ev_int_prev, rt._ev_int = getattr(rt, "_ev_int", None), ev

    def algorithmic_bytes(self) -> int:
        return 0


class StreamJoin(Op):
    """The compute stream waits for the latest edges (before a timestep's
    interior, which reads the previous edge planes, and before any other
    launch that reads the slab)."""

    family = "halo_wait"

    def __init__(self):
        self.reads = self.writes = ()

    def launch(self, rt, stream):
        ev = getattr(rt, "_ev_edges", None)
        if getattr(rt, "comm_stream", None) is None or ev is None:
            return
        import torch

        torch.cuda.current_stream(rt.device).wait_event(ev)

    def algorithmic_bytes(self) -> int:
        return 0


class EdgeOp(Op):
    """A timestep's two edge plane ranges (StarPairOps) on the communication
    stream right behind their exchange, beside the interior on the compute
    stream; they wait for the previous timestep's interior. A family of its
    own: per-launch CUDA-event timings on the compute stream do not see it."""

    family = "star_pair_edge"

    def __init__(self, edges):
        self.edges = list(edges)  # StarPairOps of the edge plane ranges
        self.reads = tuple(b for p in self.edges for b in p.reads)
        self.writes = tuple(b for p in self.edges for b in p.writes)

    def prepare(self, rt):
        for p in self.edges:
            p.prepare(rt)

    def launch(self, rt, stream):
        comm_stream = getattr(rt, "comm_stream", None)
        if comm_stream is None:
            for p in self.edges:
                p.launch(rt, stream)
            return
        import torch

        prev = getattr(rt, "_ev_int_prev", None)
        if prev is not None:
            comm_stream.wait_event(prev)
        for p in self.edges:
            p.launch(rt, comm_stream.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(comm_stream)
        rt._ev_edges = ev

    def algorithmic_bytes(self) -> int:
        return sum(p.algorithmic_bytes() for p in self.edges)


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

    solo = plan.world == 1
    ol, oh = plan.own_local
    w = plan.halo

    def pair_on(op, zr, emit=True):
        new = StarPairOp(op.a, op.b, op.fa, op.fb, op.xwrite, op.dead)
        new.X, new.Y, new.Z = loc(op.X), loc(op.Y), loc(op.Z)
        new.xout, new.zout = loc(op.xout), loc(op.zout)
        new.skip_zcopy, new.skip_xcopy = op.skip_zcopy, op.skip_xcopy
        new.plane0, new.zrange, new.global_d0 = plan.loc_lo, zr, plan.N
        new._refresh()
        if emit:
            low.emit(new)
        return new

    in_chain = False  # inside a run of timesteps (edges may be in flight)
    for op in ops:
        if isinstance(op, StarPairOp):
            if solo:
                pair_on(op, (ol, oh))
                continue
            items = [(loc(op.Y), 2)]
            if op.X.root() is not op.Y.root():
                items.append((loc(op.X), 1))
            low.emit(HaloOp(items, plan, comm, first=not in_chain))
            # interior planes read no halo plane: they overlap the exchange
            # and the edges (which follow the exchange on its stream)
            lo_edge, hi_edge = (ol, min(ol + w, oh)), (max(oh - w, ol + w), oh)
            low.emit(StreamJoin())
            if hi_edge[0] > lo_edge[1]:
                # planes per CTA 24 (the launch's own rule would pick 32):
                # measured on one rank's list, C5 at 8 ranks 21.1 -> 18.3 ms
                # per gradient, 2 and 4 ranks unchanged
                pair_on(op, (lo_edge[1], hi_edge[0])).tpm_hint = SLAB_INTERIOR_TPM
            low.emit(StreamMark())
            edges = [pair_on(op, lo_edge, emit=False)]
            if hi_edge[1] > hi_edge[0]:
                edges.append(pair_on(op, hi_edge, emit=False))
            low.emit(EdgeOp(edges))
            in_chain = True
            continue
        if in_chain:
            low.emit(StreamJoin())  # everything else runs after the edges
            in_chain = False
        if isinstance(op, ReduceOp) and op.x.root().shape == shape:
            if op.accumulate:
                raise UnsupportedConstruct("slab decomposition: accumulating reduction")
            low.emit(ReduceOp(own_view(loc(op.x)), loc(op.out), False))
            if not solo:
                low.emit(AllReduceOp(loc(op.out), comm))
        elif isinstance(op, BroadcastOp):
            low.emit(BroadcastOp(loc(op.src), op.scale, loc(op.out), op.accumulate))
        elif isinstance(op, FillOp) and op.box == whole_box(op.dst.shape):
            low.emit(FillOp(loc(op.dst), whole_box(loc(op.dst).shape), op.value))
        else:
            raise UnsupportedConstruct(f"slab decomposition does not handle '{op.family}' launches")
    if in_chain:
        low.emit(StreamJoin())
    inputs = {k: loc(b) for k, b in lw.inputs.items()}
    outputs = {k: loc(b) for k, b in lw.outputs.items()}
    seed = loc(lw.seed_buf) if lw.seed_buf is not None else None
    return DistLowered(low, inputs, outputs, seed, plan)


def torch_empty_pinned(t):
    import torch

    return torch.empty(t.shape, dtype=t.dtype, pin_memory=True)


class SlabEngine:
    """One rank of a slab-decomposed gradient: the caller's stencil program
    (any program whose fused launch list decomposes, e.g. heat_3d) over the
    ranks of a process group, one GPU per rank.

    ``step(local_inputs)`` runs on device-resident local slabs (halo planes
    included, ``local_inputs``); ``gradient(host_local_inputs)`` and
    ``gradients(batches)`` are the end-to-end calls returning the owned
    planes; ``api.gradient(..., group=...)`` wraps it for full arrays."""

    def __init__(self, program, bundle=None, params=None, *, rank=None, world=None, device=None, group=None,
                 trip_limit=None):
        import torch
        import torch.distributed as dist

        from .api import as_bundle, host_build_backward, lower_gradient
        from .ir import adopt, eval_int
        from .runtime import Executable

        self.params = dict(params or {})
        self.program = adopt(program)
        bundle = as_bundle(bundle) if bundle is not None else host_build_backward(program)
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        shapes = {n: tuple(eval_int(s, self.params) for s in d.shape)
                  for n, d in self.program.descriptors.items() if d.role == "input"}
        self.shapes = shapes
        lw = lower_gradient(self.program, bundle, self.params, shapes, fuse_small=True, trip_limit=trip_limit)
        N = next(iter(shapes.values()))[0]
        self.plan = SlabPlan(N, world, rank)
        self.dl = decompose(lw, self.plan, TorchComm(group))
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        # one rank: no communication op, so the list is captured in a CUDA
        # graph like the single-device engine; several ranks run it eagerly
        # with the exchanges on a communication stream
        # several ranks: launches on two streams, so no buffer may share
        # memory with another by liveness in list order (reuse off)
        self.exe = Executable(self.dl.low, self.dl.inputs, self.dl.outputs, seed_buf=self.dl.seed_buf,
                              device=self.device, use_graph=world == 1, reuse=world == 1)
        if world > 1:
            self.exe.comm_stream = torch.cuda.Stream(self.device)
        self.group = group

    @classmethod
    def from_workload(cls, name: str, params: dict, rank: int, world: int, device):
        from . import workloads as W

        prog, bundle = W.load(name)
        eng = cls(prog, bundle, params, rank=rank, world=world, device=device)
        eng.name = name
        return eng

    def local_slices(self, full: dict) -> dict:
        """This rank's slabs (halo planes included) of full host arrays."""
        return {k: np.ascontiguousarray(self.plan.local_slice(np.asarray(v))) for k, v in full.items()}

    def local_inputs(self, seed=0) -> dict:
        import torch

        from . import workloads as W

        full = W.make_inputs(self.name, self.program, self.params, seed)
        return {k: torch.from_numpy(v).to(self.device) for k, v in self.local_slices(full).items()}

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

    def full_gradient(self, full_inputs: dict, seed=1.0):
        """The reference call shape on every rank: full host arrays in, the
        value and the FULL gradients out (owned planes all-gathered over the
        group, so every rank returns the same arrays as the reference)."""
        import torch
        import torch.distributed as dist

        from .api import GradientResult
        from .runtime import NP_DTYPE

        res = self.gradient(self.local_slices(full_inputs), seed)
        world = self.plan.world
        grads = {}
        for ind in self.program.independents:
            desc = self.program.descriptors[ind]
            shape = self.shapes[ind]
            part = res.grads.get(ind)
            if part is None:
                grads[ind] = np.zeros(shape, dtype=NP_DTYPE[desc.element_kind])
                continue
            if world == 1:
                grads[ind] = np.array(part)
                continue
            rows = [SlabPlan(self.plan.N, world, r) for r in range(world)]
            pad = max(p.own_hi - p.own_lo for p in rows)
            mine = torch.zeros((pad,) + tuple(shape[1:]), dtype=torch.from_numpy(part).dtype, device=self.device)
            mine[:part.shape[0]].copy_(torch.from_numpy(part))
            got = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(got, mine, group=self.group)
            grads[ind] = np.concatenate([g[:p.own_hi - p.own_lo].cpu().numpy() for g, p in zip(got, rows)])
        return GradientResult(value=res.value, grads=grads, forward=None, backward=None, bundle=None)

    def own_grad(self, name: str):
        g = self.exe.output("grad:" + name)
        lo, hi = self.plan.own_local
        return g[lo:hi]
