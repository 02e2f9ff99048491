"""Executable: a lowered launch list bound to device memory.

Owns the HBM buffers of one (program(s), params) instance, prepares every
launch descriptor once, and runs the list either eagerly (first call,
programs that are not capturable) or as one captured CUDA graph replay.
Inputs are copied into engine-owned buffers on every run (the reference
copies inputs on entry and never mutates caller arrays, interpreter.py:
604-618); results are read back after one stream synchronisation, at which
point the device error word is checked and mapped to DomainError.
"""
from __future__ import annotations

import os
import weakref
from collections.abc import Mapping

import numpy as np
import torch

from . import _lib as L
from .errors import DomainError, EngineError, GradflowError
from .lowering import Buffer, Lowering

TORCH_DTYPE = {"real32": torch.float32, "real64": torch.float64}
NP_DTYPE = {"real32": np.float32, "real64": np.float64}


def require_cuda():
    if not torch.cuda.is_available():
        raise EngineError("the B200 engine needs a CUDA device; none is visible (no CPU fallback)")


def live_intervals(ops, to_end=frozenset()):
    """[first, last] launch index touching each root buffer (aliases and views
    count for their root); results stay live until read back after the run."""
    first, last = {}, {}
    for i, op in enumerate(ops):
        for b in tuple(op.reads) + tuple(op.writes):
            r = b.root().bid
            first.setdefault(r, i)
            last[r] = i
    for r in to_end:
        if r in first:
            last[r] = len(ops)
    return first, last


def memory_timeline(ops, roots, keep, to_end=frozenset(), offsets=None, buffers=()):
    """Resident bytes of the arena-placed buffers launch by launch, in the
    vocabulary of the reference ``MemoryTimeline`` (verification.py:220-226):
    events (label, delta, resident) with ``alloc <array>`` at the first
    launch that touches a buffer and ``free <array>`` after its last, plus the
    peak. Inputs, the seed and pinned buffers (the planner does not count
    them, checkpointing.py:10-17) are excluded, as in ``plan_arena``. With the
    placement ``offsets``, ``high_water`` is the highest byte addressed while
    each event holds (<= the arena size). ``aliases`` maps each placed
    buffer's name to the names of every buffer sharing its storage (copies
    the engine elides, twins), from ``buffers``."""
    first, last = live_intervals(ops, to_end)
    aliases = {}
    for b in buffers:
        aliases.setdefault(b.root().name, set()).add(b.name)
    bufs = {b.bid: b for b in roots if b.bid not in keep and b.bid in first and b.shape != ()}
    n = len(ops)
    starts, ends = {}, {}
    for bid, b in bufs.items():
        starts.setdefault(first[bid], []).append(b)
        ends.setdefault(last[bid], []).append(b)
    events, cur, peak, live = [], 0, 0, {}
    high = 0
    for i in range(n + 1):
        for b in sorted(starts.get(i, ()), key=lambda b: b.name):
            cur += b.nbytes
            live[b.bid] = b
            peak = max(peak, cur)
            if offsets is not None:
                high = max(high, offsets[b.bid] + b.nbytes)
            events.append((f"alloc {b.name}", b.nbytes, cur, i))
        for b in sorted(ends.get(i, ()), key=lambda b: b.name):
            cur -= b.nbytes
            live.pop(b.bid, None)
            events.append((f"free {b.name}", -b.nbytes, cur, i))
    return {"events": events, "peak": peak, "high_water": high,
            "aliases": {k: sorted(v) for k, v in aliases.items()}}


def plan_arena(ops, roots, keep, to_end=frozenset()):
    """Liveness-planned placement of the non-pinned root buffers in one arena:
    live interval = [first, last] launch index touching the buffer (aliases
    and views count for their root); greedy first-fit by interval start.
    Returns ({bid: byte offset}, arena bytes)."""
    first, last = live_intervals(ops, to_end)
    # scalars stay outside (the planner counts them as free, checkpointing.py:10-17)
    placed = [b for b in roots if b.bid not in keep and b.bid in first and b.shape != ()]
    # largest first, each at the lowest offset free over its whole interval
    placed.sort(key=lambda b: (-b.nbytes, first[b.bid]))
    done = []  # (offset, size, first, last)
    arena = 0
    offsets = {}
    for b in placed:
        align = 256 if b.nbytes >= 4096 else 16
        size = (max(b.nbytes, 1) + align - 1) // align * align
        f, l = first[b.bid], last[b.bid]
        busy = sorted((o, sz) for o, sz, bf, bl in done if bf <= l and f <= bl)
        off = 0
        for o, sz in busy:
            if off + size <= o:
                break
            off = max(off, (o + sz + align - 1) // align * align)
        offsets[b.bid] = off
        done.append((off, size, f, l))
        arena = max(arena, off + size)
    return offsets, arena


def _pool_only(t: torch.Tensor) -> bool:
    """True when no other tensor (e.g. the base of a numpy array made by
    ``.numpy()``, or a view) shares ``t``'s storage. Storage refs: ``t``
    itself and the temporary ``untyped_storage()`` object."""
    return torch._C._storage_Use_Count(t.untyped_storage()._cdata) <= 2


class HostEnv(Mapping):
    """``RunResult.env`` of an engine run: name -> host numpy array, copied
    from the device on first access. Before the executable runs again (which
    rewrites its buffers) every live HostEnv of it copies what it has not
    read yet, so the arrays a caller holds keep the values of their own call,
    as the reference's env does (interpreter.py:78-83)."""

    __hash__ = object.__hash__  # identity (tracked in a WeakSet); Mapping equality stays by content

    def __init__(self, exe, bufs: dict):
        self._exe, self._bufs, self._host = exe, dict(bufs), {}
        exe._live_envs.add(self)

    def __getitem__(self, name):
        got = self._host.get(name)
        if got is None:
            if name not in self._bufs:
                raise KeyError(name)
            got = self._host[name] = self._exe.view(self._bufs[name]).cpu().numpy().copy()
        return got

    def __iter__(self):
        return iter(self._bufs)

    def __len__(self):
        return len(self._bufs)

    def materialize(self):
        for name in self._bufs:
            self[name]


def _read_slots(view, groups: list) -> list:
    """Host copies of the snapshot buffers of several decisions
    ([{name: Buffer}] -> [{name: ndarray}]) with one gather and one
    device-to-host copy per element type."""
    by_kind = {}
    for gi, slots in enumerate(groups):
        for n, b in slots.items():
            by_kind.setdefault(b.kind, []).append((gi, n, b))
    out = [{} for _ in groups]
    for items in by_kind.values():
        flat = torch.cat([view(b).reshape(-1) for _, _, b in items]).cpu().numpy()
        o = 0
        for gi, n, b in items:
            out[gi][n] = flat[o:o + b.numel].reshape(b.shape)
            o += b.numel
    return out


class ProbeRuntime:
    """Incremental executor for the data-dependent decisions met while a
    launch list is lowered (reference branches and scalar loop headers,
    interpreter.py:210-219, 342-347). At each decision it runs only the
    launches emitted since the previous one, on buffers it keeps for the
    whole lowering (one allocation per buffer, no arena reuse), and reads
    the decision's snapshots back: T decisions cost O(T) launches, where
    lowering again from the start for every decision cost O(T^2). Buffer
    tensors are bound only while its launches are prepared and run, so the
    final Executable plans its own arena."""

    def __init__(self, inputs: dict, seed=1.0, device=None):
        require_cuda()
        self.lib = L.load()
        self.device = torch.device(device or "cuda")
        self.inputs = inputs
        self.seed = seed
        self.tensors = {}  # root bid -> tensor
        self.done = 0      # launches already run
        self.loaded = False
        self.seeded = False
        self.aux = []
        self.workspace = torch.empty(16, dtype=torch.uint8, device=self.device)
        self.workspace_ptr = self.workspace.data_ptr()
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.err_ptr = self.err.data_ptr()
        self.launches = 0

    def upload(self, arr: np.ndarray) -> int:
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(self.device)
        self.aux.append(t)
        return t.data_ptr()

    def view(self, b: Buffer) -> torch.Tensor:
        t = self.tensors[b.root().bid]
        o = b.root_offset()
        return t[o: o + b.numel].view(b.shape) if b.shape else t[o:o + 1].view(())

    def __call__(self, low: Lowering, slots: dict) -> dict:
        roots = {}
        for b in low.buffers:
            r = b.root()
            if r.tensor is not None and r.bid not in self.tensors:
                continue  # placed by its owner (not this prober's to bind or release)
            roots[r.bid] = r
            if r.bid not in self.tensors:
                self.tensors[r.bid] = torch.empty(max(r.numel, 1), dtype=TORCH_DTYPE[r.kind], device=self.device)
        for bid, r in roots.items():
            r.tensor = self.tensors[bid]
        try:
            if not self.loaded:
                for name, buf in low.entry_inputs.items():
                    v = self.inputs[name]
                    dst = self.view(buf)
                    src = v if isinstance(v, torch.Tensor) else torch.from_numpy(
                        np.ascontiguousarray(np.asarray(v, dtype=NP_DTYPE[buf.kind])))
                    dst.copy_(src.reshape(dst.shape).to(dst.dtype))
                self.loaded = True
            if getattr(low, "entry_seed", None) is not None and not self.seeded:
                self.view(low.entry_seed).fill_(float(self.seed))
                self.seeded = True
            new = low.ops[self.done:]
            ws = max([int(op.workspace_bytes()) for op in new if hasattr(op, "workspace_bytes")] + [16])
            if ws > self.workspace.numel():
                self.workspace = torch.empty(ws, dtype=torch.uint8, device=self.device)
                self.workspace_ptr = self.workspace.data_ptr()
            stream = torch.cuda.current_stream(self.device).cuda_stream
            for op in new:
                op.prepare(self)
                op.launch(self, stream)
            self.launches += len(new)
            self.done = len(low.ops)
            torch.cuda.synchronize(self.device)
            bits = int(self.err.item())
            if bits:
                msgs = [m for b_, m in L.EBITS.items() if bits & b_]
                raise DomainError("; ".join(msgs) or f"device error bits {bits:#x}")
            return {n: v.copy() for n, v in _read_slots(self.view, [slots])[0].items()}
        finally:
            for r in roots.values():
                r.tensor = None


class Executable:
    def __init__(self, low: Lowering, inputs: dict, outputs: dict, *, seed_buf: Buffer | None = None,
                 device=None, use_graph: bool | None = None, pinned=(), reuse: bool | None = None):
        require_cuda()
        self.lib = L.load()
        self.low = low
        self.ops = low.ops
        self.inputs = inputs      # caller name -> Buffer
        self.outputs = outputs    # key -> Buffer
        self.seed_buf = seed_buf
        self.device = torch.device(device or "cuda")
        self.flops = low.flops
        env_graph = os.environ.get("GFB_GRAPH", "1") != "0"
        self.use_graph = env_graph if use_graph is None else use_graph
        self.graph = None
        self.runs = 0
        # decision snapshots (data-dependent control flow) stay readable
        self.pinned = list(pinned) + [low.resolve(b) for slots, _, _ in low.decisions for b in slots.values()]
        self.reuse = (os.environ.get("GFB_ARENA", "1") != "0") if reuse is None else reuse
        self._live_envs = weakref.WeakSet()
        self._allocate()
        for op in self.ops:
            op.prepare(self)

    # -- memory ------------------------------------------------------------------

    def _allocate(self):
        """Place every root buffer. With reuse (default), buffers that are not
        live at the same time share one liveness-planned HBM arena (first-fit
        over [first use, last use] intervals of the launch list); inputs,
        outputs, the seed and explicitly pinned buffers live for the whole
        run. ``payload_peak`` is the arena size: the device-side counterpart
        of the planner's peak (checkpointing.py:10-17 counts intermediates,
        gradients and kept values, not inputs or the dependent)."""
        roots = [b for b in self.low.buffers if b.alias_of is None and b.tensor is None]
        keep = {b.root().bid for b in list(self.inputs.values()) + self.pinned}
        if self.seed_buf is not None:
            keep.add(self.seed_buf.root().bid)
        outs = {b.root().bid for b in self.outputs.values()}
        offsets, arena = plan_arena(self.ops, roots, keep, outs) if self.reuse else ({}, 0)
        self._placement = (roots, keep, outs, offsets)
        total = 0
        placed = [b for b in roots if b.bid in offsets]
        for b in roots:
            if b.bid not in offsets:
                b.tensor = torch.empty(max(b.numel, 1), dtype=TORCH_DTYPE[b.kind], device=self.device)
                total += b.tensor.numel() * b.tensor.element_size()
        self.arena = torch.empty(max(arena, 256), dtype=torch.uint8, device=self.device)
        self.keep_bids = keep
        for b in placed:
            o = offsets[b.bid]
            b.tensor = self.arena[o:o + max(b.nbytes, 1) + (-max(b.nbytes, 1)) % b.itemsize].view(TORCH_DTYPE[b.kind])
        self.payload_peak = arena
        self.keep_bids = keep | outs | {b.bid for b in roots if b.tensor is not None and b.bid not in offsets}
        total += arena
        ws = 0
        for op in self.ops:
            f = getattr(op, "workspace_bytes", None)
            if f is not None:
                ws = max(ws, int(f()))
        self.workspace = torch.empty(max(ws, 16), dtype=torch.uint8, device=self.device)
        self.workspace_ptr = self.workspace.data_ptr()
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.err_ptr = self.err.data_ptr()
        self.aux = []  # static per-launch tables (index tables of contractions)
        self.device_bytes = total + self.workspace.numel()

    def memory_timeline(self) -> dict:
        """Arena residency launch by launch (``memory_timeline``) of this
        executable's actual placement."""
        roots, keep, outs, offsets = self._placement
        return memory_timeline(self.ops, roots, keep, outs, offsets if offsets else None, self.low.buffers)

    def upload(self, arr: np.ndarray) -> int:
        """Copy a static host table to device memory owned by this executable;
        returns its device pointer."""
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(self.device)
        self.aux.append(t)
        self.device_bytes += t.numel() * t.element_size()
        return t.data_ptr()

    def view(self, b: Buffer) -> torch.Tensor:
        t = b.root().tensor
        o = b.root_offset()
        return t[o: o + b.numel].view(b.shape) if b.shape else t[o:o + 1].view(())

    # -- execution -----------------------------------------------------------------

    def load_inputs(self, values: dict):
        for name, buf in self.inputs.items():
            v = values[name]
            dst = self.view(buf)
            if isinstance(v, torch.Tensor):
                src = v if v.dtype == dst.dtype else v.to(dst.dtype)
                if tuple(src.shape) != tuple(dst.shape):
                    src = src.reshape(dst.shape)
                # device tensors: one D2D copy; pinned host tensors: async DMA
                dst.copy_(src, non_blocking=True)
            else:
                arr = np.ascontiguousarray(np.asarray(v, dtype=NP_DTYPE[buf.kind])).reshape(buf.shape)
                dst.copy_(torch.from_numpy(arr), non_blocking=False)

    def launch_all(self):
        stream = torch.cuda.current_stream(self.device).cuda_stream
        if self.graph is not None:
            self.graph.replay()
            return
        for op in self.ops:
            op.launch(self, stream)

    def run(self, inputs: dict, seed=1.0, *, sync=True, clear_err=True):
        for env in list(self._live_envs):
            env.materialize()  # results of the previous call keep their values
        self._live_envs.clear()
        self.load_inputs(inputs)
        if self.seed_buf is not None:
            self.view(self.seed_buf).fill_(float(seed))
        if clear_err:
            self.err.zero_()
        if self.graph is None and self.use_graph and self.runs >= 1:
            self._capture()
        self.launch_all()
        self.runs += 1
        if sync:
            self.check()

    def _capture(self):
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize(self.device)
        with torch.cuda.graph(g):
            stream = torch.cuda.current_stream(self.device).cuda_stream
            for op in self.ops:
                op.launch(self, stream)
        self.graph = g

    def check(self):
        torch.cuda.synchronize(self.device)
        bits = int(self.err.item())
        if bits:
            msgs = [m for b, m in L.EBITS.items() if bits & b]
            raise DomainError("; ".join(msgs) or f"device error bits {bits:#x}")

    def decisions_hold(self) -> bool:
        """Re-evaluate every data-dependent control-flow decision this launch
        list was lowered with, from the device snapshots of the run just
        finished; False means the inputs took another path and the caller
        must lower again."""
        # one device-to-host copy per element type for all snapshots
        host = _read_slots(self.view, [{n: self.low.resolve(b) for n, b in slots.items()}
                                       for slots, _k, _v in self.low.decisions])
        for vals, (_slots, key_fn, key) in zip(host, self.low.decisions):
            try:
                if key_fn(vals) != key:
                    return False
            except GradflowError:
                # a later decision's snapshot taken along the stale path can
                # be out of its domain (e.g. a non-integer loop header): the
                # path changed earlier, so lower again
                return False
        return True

    def _host_slot(self, like: dict) -> dict:
        """Pinned host result tensors shaped like ``like``, from a pool owned
        by this executable: an entry is reused once nothing outside the pool
        references its tensors (results handed to the caller keep theirs).
        A fresh 1 GiB pinned allocation costs ~0.8 s (cudaHostAlloc), longer
        than five C5 steps. An entry stays busy while its step is in flight;
        once yielded, the caller's ``.numpy()`` arrays (or any view) hold it."""
        sig = tuple((k, tuple(t.shape), t.dtype) for k, t in like.items())
        pool = self.__dict__.setdefault("_host_pool", [])
        busy = self.__dict__.setdefault("_host_busy", set())
        for s_, entry in pool:
            if s_ == sig and id(entry) not in busy and all(_pool_only(t) for t in entry.values()):
                busy.add(id(entry))
                return entry
        entry = {k: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for k, t in like.items()}
        pool.append((sig, entry))
        busy.add(id(entry))
        return entry

    def run_pipelined(self, batches, outputs: dict, seed=1.0):
        """End-to-end runs over an iterable of input dicts (pinned host
        tensors for asynchronous DMA), overlapped across steps: while step k
        computes, the copy engines move step k+1's inputs in and step k-1's
        results out (PCIe is full duplex; the launch list owns one set of
        input buffers, so inputs land in one of two device staging slots and
        enter the launch list by a device copy, ~0.5 % of a C5 step).

        ``outputs`` maps result keys to device views of this executable's
        buffers (``output(key)`` or a slice of it). Yields one dict per batch,
        in order, of fresh pinned host tensors, after checking that step's
        device error word (``DomainError``). The yielded tensors are pooled
        pinned memory: take ``.numpy()`` (or a view / clone) before requesting
        the next result; that array keeps the slot from being reused."""
        from collections import deque

        dev = self.device
        comp = torch.cuda.current_stream(dev)
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        names = list(self.inputs)
        dst_in = {n: self.view(self.inputs[n]) for n in names}
        src_out = dict(outputs)
        src_out["#err"] = self.err
        stage_in = [{n: torch.empty_like(t) for n, t in dst_in.items()} for _ in range(2)]
        stage_out = [{k: torch.empty_like(t) for k, t in src_out.items()} for _ in range(2)]
        ev = lambda: [torch.cuda.Event(), torch.cuda.Event()]  # noqa: E731
        in_ready, in_free, out_ready, out_free = ev(), ev(), ev(), ev()
        if self.graph is None and self.use_graph and self.runs >= 1:
            self._capture()
        pending = deque()

        def finish(item):
            done, host, slot = item
            done.synchronize()
            self._host_busy.discard(id(slot))
            bits = int(host.pop("#err").item())
            if bits:
                msgs = [m for b, m in L.EBITS.items() if bits & b]
                raise DomainError("; ".join(msgs) or f"device error bits {bits:#x}")
            return host

        try:
            for k, batch in enumerate(batches):
                j = k & 1
                s_in.wait_event(in_free[j])
                with torch.cuda.stream(s_in):
                    for n in names:
                        v = batch[n]
                        if not isinstance(v, torch.Tensor):
                            v = torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=NP_DTYPE[self.inputs[n].kind])))
                        stage_in[j][n].copy_(v.reshape(stage_in[j][n].shape), non_blocking=True)
                    in_ready[j].record(s_in)
                comp.wait_event(in_ready[j])
                for n in names:
                    dst_in[n].copy_(stage_in[j][n], non_blocking=True)
                in_free[j].record(comp)
                if self.seed_buf is not None:
                    self.view(self.seed_buf).fill_(float(seed))
                self.err.zero_()
                self.launch_all()
                self.runs += 1
                comp.wait_event(out_free[j])
                for key, t in src_out.items():
                    stage_out[j][key].copy_(t, non_blocking=True)
                out_ready[j].record(comp)
                s_out.wait_event(out_ready[j])
                with torch.cuda.stream(s_out):
                    slot = self._host_slot(src_out)
                    host = dict(slot)
                    for key in src_out:
                        host[key].copy_(stage_out[j][key], non_blocking=True)
                    out_free[j].record(s_out)
                    done = torch.cuda.Event()
                    done.record(s_out)
                pending.append((done, host, slot))
                if len(pending) > 1:
                    yield finish(pending.popleft())
            while pending:
                yield finish(pending.popleft())
        finally:  # an abandoned generator releases its in-flight slots
            for _, _, slot in pending:
                self._host_busy.discard(id(slot))

    def output(self, key) -> torch.Tensor:
        return self.view(self.outputs[key])

    def output_host(self, key) -> np.ndarray:
        """Fresh host array (owned by the caller) via a pinned staging copy."""
        t = self.output(key)
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return h.numpy()

    # -- profiling helpers ----------------------------------------------------------

    def timed_eager(self, inputs: dict, seed=1.0):
        """One eager run with a CUDA event pair around every launch; returns
        [(family, op, ms)] (used by bench.py for per-kernel roofline shares)."""
        self.load_inputs(inputs)
        if self.seed_buf is not None:
            self.view(self.seed_buf).fill_(float(seed))
        self.err.zero_()
        stream = torch.cuda.current_stream(self.device)
        evs = []
        # hold the stream with a device-side spin while the host enqueues every
        # launch, so each event pair brackets GPU execution only (not the
        # host's per-launch latency); ~40 us of host time per launch
        torch.cuda._sleep(int(min(len(self.ops) * 40e-6, 2.0) * 2e9))
        for op in self.ops:
            if getattr(op, "elided", False):
                continue  # an alias, not a launch
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            op.launch(self, stream.cuda_stream)
            b.record(stream)
            evs.append((op, a, b))
        self.check()
        return [(op.family, op, a.elapsed_time(b)) for op, a, b in evs]
