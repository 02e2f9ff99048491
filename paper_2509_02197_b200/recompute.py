"""Recompute fused into the adjoint kernels that consume it.

A plan (reference ``plan()``, checkpointing.py:852-900) that recomputes a
forwarded value V splices a ``rec_<name>`` block before its first use in the
reverse program (``apply_plan``, checkpointing.py:813-821; the block is the
replayed producer chain built by ``_recompute_plan``, :345-442). Executed
literally, every stage of the block is a launch that writes a full array to
HBM, which the adjoint map then reads back.

This pass rewrites the reverse program before lowering so that the
elementwise stages of a recompute block are evaluated inside the consuming
adjoint kernels instead:

* a producer is an elementwise stage of a ``rec_*`` state whose output V is
  a rank >= 1 temporary written nowhere else: an ``ew_unary`` / ``ew_binary``
  library node (reference interpreter.py:553-597), or a single-tasklet map
  writing V at exactly its own parameters (identity, no ``wcr``);
* every read of V elsewhere in the program is an input connector of a map
  tasklet (or a state-level tasklet) at some subset s; V[s] is replaced by
  the producer's expression with its own subsets composed with s (V[p] =
  f(X[sigma(p)]) gives V[s] = f(X[sigma(s)]));
* the producer's inputs are never written after the producer (forward
  inputs, or earlier temporaries of the same block), so the consumer sees
  the values the block would have used;
* only operations that cannot raise a domain error are inlined (no div,
  log, sqrt, pow, idiv, mod): the reference evaluates the block for every
  element eagerly (symexpr.py:81-133), and an inlined copy evaluates only
  the elements the consumer reads.

Chains fuse from the consumer back (r1 = relu(h1 + b1): both maps fold into
the adjoint body; the matmul that produces the operand stays a launch).
A state left without computing nodes disappears, so a block that is wholly
elementwise (softmax ``rec_e__v1 = exp(x)``) costs no launch and no HBM
array at all. Values, gradients and the planner's decisions are unchanged;
the device peak can only go down (tests/test_gpu_r2.py pins both).
"""
from __future__ import annotations

import copy

from .ir import (
    AccessNode,
    Binary,
    Conditional,
    Const,
    Dataflow,
    Index,
    LibraryNode,
    LoopRegion,
    MapNode,
    Memlet,
    Name,
    Program,
    State,
    Tasklet,
    Unary,
    walk_blocks,
)

SAFE_UNARY = {"neg", "sin", "cos", "exp", "tanh", "abs", "sign"}
SAFE_BINARY = {"add", "sub", "mul", "min", "max"}
LIB_UNARY = {"copy", "scale", "neg", "abs", "sign", "sin", "cos", "exp", "tanh"}
LIB_BINARY = {"add", "sub", "mul", "min", "max"}


def _safe(expr) -> bool:
    t = type(expr)
    if t in (Const, Name):
        return True
    if t is Unary:
        return expr.op in SAFE_UNARY and _safe(expr.x)
    if t is Binary:
        return expr.op in SAFE_BINARY and _safe(expr.x) and _safe(expr.y)
    return False


def _subst(expr, env: dict):
    """Replace Name(k) by env[k] (expressions)."""
    t = type(expr)
    if t is Name:
        return env.get(expr.id, expr)
    if t is Unary:
        return Unary(expr.op, _subst(expr.x, env))
    if t is Binary:
        return Binary(expr.op, _subst(expr.x, env), _subst(expr.y, env))
    if t is Index:
        return Index(expr.base, tuple(_subst(e, env) for e in expr.indices))
    return expr


def _writes(program: Program) -> dict:
    """data -> number of write edges (into an access node) in the program."""
    out = {}
    for _, b in walk_blocks(program.region):
        if isinstance(b, State):
            access = {n.id for n in b.graph.nodes if isinstance(n, AccessNode)}
            for e in b.graph.edges:
                if e.dst in access:
                    out[e.data] = out.get(e.data, 0) + 1
    return out


class _Producer:
    """V = f(inputs): ``inputs`` = [(connector, data, subset over params or
    None for same-shape library operands)], ``body`` over the connectors."""

    def __init__(self, state, node, out_access, data, params, inputs, body):
        self.state, self.node, self.out_access, self.data = state, node, out_access, data
        self.params, self.inputs, self.body = params, inputs, body


def _producers(program: Program, writes: dict, protected: set):
    for _, b in walk_blocks(program.region):
        if not (isinstance(b, State) and b.label.startswith("rec_")):
            continue
        g = b.graph
        for n in g.nodes:
            if isinstance(n, AccessNode):
                continue
            outs = g.out_edges(n.id)
            if len(outs) != 1 or outs[0].wcr is not None:
                continue
            v = outs[0].data
            desc = program.descriptors.get(v)
            if desc is None or desc.rank == 0 or writes.get(v, 0) != 1 or v in protected:
                continue
            ins = g.in_edges(n.id)
            if isinstance(n, LibraryNode):
                if n.kind == "ew_unary" and n.op in LIB_UNARY and len(ins) == 1:
                    x = Name("x")
                    body = {"copy": x, "scale": Binary("mul", Const(float(n.const or 0.0)), x)}.get(n.op)
                    body = body if body is not None else Unary(n.op, x)
                elif n.kind == "ew_binary" and n.op in LIB_BINARY and len(ins) == 2:
                    body = Binary(n.op, Name("a"), Name("b"))
                else:
                    continue
                # library operands have V's shape: element-for-element
                if any(program.descriptors[e.data].shape != desc.shape for e in ins):
                    continue
                yield _Producer(b, n, outs[0].dst, v, None, [(e.dst_conn, e.data, None) for e in ins], body)
            elif isinstance(n, MapNode):
                computes = [m for m in n.body.nodes if not isinstance(m, AccessNode)]
                if len(computes) != 1 or not isinstance(computes[0], Tasklet):
                    continue
                t = computes[0]
                bouts = n.body.out_edges(t.id)
                if len(bouts) != 1 or bouts[0].wcr is not None or bouts[0].data != v:
                    continue
                # V written at exactly the map parameters over V's full extent
                if tuple(bouts[0].subset or ()) != tuple(Name(p) for p in n.params):
                    continue
                if len(n.params) != desc.rank or any(
                        r[0] != Const(0) or r[1] != s or r[2] != Const(1) for r, s in zip(n.ranges, desc.shape)):
                    continue
                body = t.body[bouts[0].src_conn]
                bins = n.body.in_edges(t.id)
                yield _Producer(b, n, outs[0].dst, v, tuple(n.params),
                                [(e.dst_conn, e.data, tuple(e.subset or ())) for e in bins], body)


def _consumers(program: Program, v: str):
    """Every read of v: (state, tasklet, map node or None, graph, edge); None
    if some read is not a tasklet input connector."""
    found = []
    for _, b in walk_blocks(program.region):
        if not isinstance(b, State):
            continue
        g = b.graph
        for e in g.edges:
            if e.data != v:
                continue
            src = g.node(e.src)
            dst = g.node(e.dst)
            if isinstance(src, AccessNode) and isinstance(dst, MapNode):
                continue  # the map's outer edge; its body edges are checked below
            if isinstance(src, AccessNode) and isinstance(dst, Tasklet):
                found.append((b, dst, None, g, e))
            elif isinstance(dst, AccessNode) and isinstance(src, (Tasklet, MapNode, LibraryNode)):
                continue  # the write (the producer)
            else:
                return None
        for n in g.nodes:
            if isinstance(n, MapNode):
                for e in n.body.edges:
                    if e.data == v:
                        dst = n.body.node(e.dst)
                        if not isinstance(dst, Tasklet) or e.dst_conn is None:
                            return None
                        found.append((b, dst, n, n.body, e))
    return found


def fuse_recompute(program: Program):
    """(rewritten program, [fused value names]). The input program is not
    modified."""
    prog = copy.deepcopy(program)
    protected = set(prog.independents) | {prog.dependent} | {
        d.name for d in prog.descriptors.values() if d.role in ("input", "output")}
    fused = []
    while True:
        writes = _writes(prog)
        done = False
        for pr in _producers(prog, writes, protected):
            # inputs unchanged between producer and consumers: written at
            # most once (an earlier stage of the block) or never
            if any(writes.get(d, 0) > 1 for _, d, _ in pr.inputs):
                continue
            cons = _consumers(prog, pr.data)
            if not cons or not _safe(pr.body) or any(e.dst_conn not in t.ins for _, t, _, _, e in cons):
                continue
            for c in cons:
                _inline(prog, pr, c)
            _remove_producer(prog, pr)
            fused.append(pr.data)
            done = True
            break
        if not done:
            break
    _drop_empty_states(prog.region)
    return prog, fused


def _inline(prog: Program, pr: _Producer, c):
    state, t, mnode, g, e = c
    conn = e.dst_conn
    s = tuple(e.subset or ())
    env_idx = dict(zip(pr.params, s)) if pr.params is not None else None
    new_names = {}
    for k, data, sub in pr.inputs:
        nc = f"{conn}__{k}"
        while nc in t.ins or nc in t.outs:
            nc += "_"
        new_names[k] = Name(nc)
        if pr.params is None:
            nsub = s  # same-shape library operand: element-for-element
        else:
            nsub = tuple(_subst(x, env_idx) for x in sub)
        # an access node of the operand in the consumer's graph
        aid = f"{e.src}__rc_{nc}"
        g.nodes.append(AccessNode(aid, data))
        g.edges.append(Memlet(aid, None, t.id, nc, data, nsub))
        t.ins = tuple(t.ins) + (nc,)
        if mnode is not None:
            # and an outer edge into the map: from the state's instance of the
            # operand that holds its value here (the last written one when
            # the operand is produced in this state, e.g. by an earlier stage
            # of the same recompute block), else a fresh read-only instance
            outer = state.graph
            inst = [n.id for n in outer.nodes if isinstance(n, AccessNode) and n.data == data]
            written = [i for i in inst if outer.in_edges(i)]
            if written:
                oid = written[-1]
            elif inst:
                oid = inst[0]
            else:
                oid = f"{mnode.id}__rc_{nc}"
                outer.nodes.insert(0, AccessNode(oid, data))
            outer.edges.append(Memlet(oid, None, mnode.id, None, data, None))
    expr = _subst(pr.body, new_names)
    t.body = {k: _subst(v, {conn: expr}) for k, v in t.body.items()}
    t.ins = tuple(x for x in t.ins if x != conn)
    g.edges.remove(e)
    src = e.src
    if not any(x.src == src or x.dst == src for x in g.edges):
        g.nodes = [n for n in g.nodes if n.id != src]
    if mnode is not None:
        outer = state.graph
        if not any(x.data == pr.data for x in mnode.body.edges):
            for oe in [x for x in outer.edges if x.dst == mnode.id and x.data == pr.data]:
                outer.edges.remove(oe)
                if not any(x.src == oe.src or x.dst == oe.src for x in outer.edges):
                    outer.nodes = [n for n in outer.nodes if n.id != oe.src]


def _remove_producer(prog: Program, pr: _Producer):
    g = pr.state.graph
    g.edges = [e for e in g.edges if e.src != pr.node.id and e.dst != pr.node.id]
    g.nodes = [n for n in g.nodes if n.id not in (pr.node.id, pr.out_access)]
    used = {e.src for e in g.edges} | {e.dst for e in g.edges}
    g.nodes = [n for n in g.nodes if not isinstance(n, AccessNode) or n.id in used]


def _drop_empty_states(region: list):
    keep = []
    for b in region:
        if isinstance(b, State):
            if b.label.startswith("rec_") and not any(not isinstance(n, AccessNode) for n in b.graph.nodes):
                continue
        elif isinstance(b, LoopRegion):
            _drop_empty_states(b.body)
        elif isinstance(b, Conditional):
            _drop_empty_states(b.then_body)
            _drop_empty_states(b.else_body)
        keep.append(b)
    region[:] = keep


__all__ = ["fuse_recompute", "Dataflow"]
