"""Program IR consumed by the B200 engine.

The engine executes the programs that the reference AD emits
(``gradflow``; data model in reference ``pkg/src/gradflow/ir.py:50-219``,
expressions in ``symexpr.py:34-65``). This module carries an independent
implementation of that data model with the same field names, so that

* reference ``Program`` objects are adopted structurally (``adopt``) without
  importing the reference, and
* the reference's JSON wire format (``format_version`` 1, reference
  ``frontend.py:37-397``) is read and written here (``load_program``,
  ``dump_program``), which is how programs reach a GPU box that has no
  reference installation.

Only what the executor needs lives here: expression evaluation over integer
bindings, the per-state schedule (identical tie-breaking to reference
``ir.py:253-306``) and write-version numbering (reference
``versions.py:82-105``).
"""
from __future__ import annotations

import heapq
import json
import math
import re
from dataclasses import dataclass, field
from typing import Union

from .errors import DomainError, ProgramSyntaxError, UnboundName, UnsupportedLoop

# ---------------------------------------------------------------------------
# expressions


@dataclass(frozen=True)
class Const:
    value: Union[int, float]


@dataclass(frozen=True)
class Name:
    id: str


@dataclass(frozen=True)
class Unary:
    op: str
    x: "Expr"


@dataclass(frozen=True)
class Binary:
    op: str
    x: "Expr"
    y: "Expr"


@dataclass(frozen=True)
class Index:
    base: str
    indices: tuple


Expr = Union[Const, Name, Unary, Binary, Index]

BINARY_OPS = ("add", "sub", "mul", "div", "idiv", "mod", "min", "max", "pow")
UNARY_OPS = ("neg", "sin", "cos", "exp", "log", "sqrt", "tanh", "abs", "sign")
COMPARE_OPS = ("lt", "gt", "le", "ge")


def _py_div(a, b):
    if b == 0:
        raise DomainError("division by zero")
    return a / b


def _py_idiv(a, b):
    if b == 0:
        raise DomainError("floor division by zero")
    return a // b


def _py_mod(a, b):
    if b == 0:
        raise DomainError("modulo by zero")
    return a % b


def _py_pow(a, b):
    if a == 0 and b < 0:
        raise DomainError("pow: zero base with negative exponent")
    if a < 0 and not float(b).is_integer():
        raise DomainError("pow: negative base with fractional exponent")
    return a**b


def _py_log(x):
    if x <= 0:
        raise DomainError("log of non-positive value")
    return math.log(x)


def _py_sqrt(x):
    if x < 0:
        raise DomainError("sqrt of negative value")
    return math.sqrt(x)


_BIN = {
    "add": lambda a, b: a + b,
    "sub": lambda a, b: a - b,
    "mul": lambda a, b: a * b,
    "div": _py_div,
    "idiv": _py_idiv,
    "mod": _py_mod,
    "min": lambda a, b: b if b < a else a,
    "max": lambda a, b: b if b > a else a,
    "pow": _py_pow,
    "lt": lambda a, b: a < b,
    "gt": lambda a, b: a > b,
    "le": lambda a, b: a <= b,
    "ge": lambda a, b: a >= b,
}
_UN = {
    "neg": lambda x: -x,
    "sin": math.sin,
    "cos": math.cos,
    "exp": math.exp,
    "log": _py_log,
    "sqrt": _py_sqrt,
    "tanh": math.tanh,
    "abs": abs,
    "sign": lambda x: 0 if x == 0 else (1 if x > 0 else -1),
}


def evaluate(expr: Expr, bind: dict, index_fn=None):
    """Scalar evaluation (reference ``eval_expr``, symexpr.py:165-185).
    ``index_fn(base, idx_tuple)`` backs ``idx`` reads in conditions."""
    t = type(expr)
    if t is Const:
        return expr.value
    if t is Name:
        try:
            return bind[expr.id]
        except KeyError:
            raise UnboundName(f"no binding for '{expr.id}'") from None
    if t is Binary:
        return _BIN[expr.op](evaluate(expr.x, bind, index_fn), evaluate(expr.y, bind, index_fn))
    if t is Unary:
        return _UN[expr.op](evaluate(expr.x, bind, index_fn))
    if t is Index:
        if index_fn is None:
            raise UnboundName(f"no array available for '{expr.base}'")
        return index_fn(expr.base, tuple(int(evaluate(e, bind, index_fn)) for e in expr.indices))
    raise TypeError(f"not an expression: {expr!r}")


def eval_int(expr: Expr, bind: dict, what: str = "expression") -> int:
    v = evaluate(expr, bind)
    f = float(v)
    if not f.is_integer():
        raise DomainError(f"{what} evaluated to non-integer {f}")
    return int(f)


def free_names(expr: Expr) -> set:
    t = type(expr)
    if t is Const:
        return set()
    if t is Name:
        return {expr.id}
    if t is Unary:
        return free_names(expr.x)
    if t is Binary:
        return free_names(expr.x) | free_names(expr.y)
    if t is Index:
        out = {expr.base}
        for e in expr.indices:
            out |= free_names(e)
        return out
    raise TypeError(f"not an expression: {expr!r}")


def count_ops(expr: Expr) -> int:
    """Operator applications (the FLOP unit of reference symexpr.py:233-243)."""
    t = type(expr)
    if t in (Const, Name):
        return 0
    if t is Unary:
        return 1 + count_ops(expr.x)
    if t is Binary:
        return 1 + count_ops(expr.x) + count_ops(expr.y)
    if t is Index:
        return sum(count_ops(e) for e in expr.indices)
    raise TypeError(f"not an expression: {expr!r}")


_TOK = re.compile(r"\(|\)|[^\s()]+")
_IDENT = re.compile(r"^[A-Za-z_][A-Za-z0-9_]*$")


def parse_sexpr(text: str) -> Expr:
    toks = _TOK.findall(text)
    pos = 0

    def atom(tok):
        try:
            return Const(int(tok))
        except ValueError:
            pass
        try:
            return Const(float(tok))
        except ValueError:
            pass
        if _IDENT.match(tok):
            return Name(tok)
        raise ProgramSyntaxError(f"bad token '{tok}' in '{text}'")

    def one():
        nonlocal pos
        if pos >= len(toks):
            raise ProgramSyntaxError(f"unexpected end of '{text}'")
        tok = toks[pos]
        pos += 1
        if tok == ")":
            raise ProgramSyntaxError(f"unexpected ')' in '{text}'")
        if tok != "(":
            return atom(tok)
        head = toks[pos]
        pos += 1
        if head == "idx":
            base = toks[pos]
            pos += 1
            args = []
            while toks[pos] != ")":
                args.append(one())
            pos += 1
            return Index(base, tuple(args))
        args = []
        while pos < len(toks) and toks[pos] != ")":
            args.append(one())
        if pos >= len(toks):
            raise ProgramSyntaxError(f"unclosed '(' in '{text}'")
        pos += 1
        if head in UNARY_OPS and len(args) == 1:
            return Unary(head, args[0])
        if (head in BINARY_OPS or head in COMPARE_OPS) and len(args) == 2:
            return Binary(head, args[0], args[1])
        raise ProgramSyntaxError(f"bad operator '{head}' in '{text}'")

    out = one()
    if pos != len(toks):
        raise ProgramSyntaxError(f"trailing input in '{text}'")
    return out


def to_sexpr(expr: Expr) -> str:
    t = type(expr)
    if t is Const:
        v = expr.value
        return str(v) if isinstance(v, int) and not isinstance(v, bool) else repr(float(v))
    if t is Name:
        return expr.id
    if t is Unary:
        return f"({expr.op} {to_sexpr(expr.x)})"
    if t is Binary:
        return f"({expr.op} {to_sexpr(expr.x)} {to_sexpr(expr.y)})"
    if t is Index:
        return f"(idx {expr.base} " + " ".join(to_sexpr(e) for e in expr.indices) + ")"
    raise TypeError(f"not an expression: {expr!r}")


# ---------------------------------------------------------------------------
# dataflow + control flow


@dataclass(frozen=True)
class DataDescriptor:
    name: str
    element_kind: str
    shape: tuple
    role: str

    @property
    def rank(self) -> int:
        return len(self.shape)


@dataclass
class AccessNode:
    id: str
    data: str


@dataclass
class Tasklet:
    id: str
    ins: tuple
    outs: tuple
    body: dict
    group: str | None = None


@dataclass
class LibraryNode:
    id: str
    kind: str
    op: str | None = None
    const: float | None = None
    ta: bool = False
    tb: bool = False
    group: str | None = None


@dataclass
class MapNode:
    id: str
    params: tuple
    ranges: tuple
    body: "Dataflow"
    group: str | None = None


@dataclass
class Memlet:
    src: str
    src_conn: str | None
    dst: str
    dst_conn: str | None
    data: str
    subset: tuple | None
    wcr: str | None = None


@dataclass
class Dataflow:
    nodes: list = field(default_factory=list)
    edges: list = field(default_factory=list)

    def node(self, nid: str):
        for n in self.nodes:
            if n.id == nid:
                return n
        raise KeyError(nid)

    def in_edges(self, nid: str) -> list:
        return [e for e in self.edges if e.dst == nid]

    def out_edges(self, nid: str) -> list:
        return [e for e in self.edges if e.src == nid]


@dataclass
class State:
    label: str
    graph: Dataflow = field(default_factory=Dataflow)


@dataclass
class LoopRegion:
    label: str
    iterator: str
    init: Expr
    bound: Expr
    cmp: str
    update: Expr
    body: list = field(default_factory=list)
    inverse: Expr | None = None
    reversed_simulate: bool = False
    replay_of: str | None = None
    reverse_of: str | None = None


@dataclass
class Conditional:
    label: str
    condition: Expr
    then_body: list = field(default_factory=list)
    else_body: list = field(default_factory=list)
    trace_ref: str | None = None


@dataclass
class Program:
    descriptors: dict
    parameters: tuple
    region: list
    dependent: str
    independents: tuple


@dataclass(frozen=True)
class Candidate:
    version: int
    directives: tuple = ()


@dataclass(frozen=True)
class ForwardingEntry:
    name: str
    data: str
    candidates: tuple


def walk_blocks(region, path=()):
    for b in region:
        yield path, b
        if isinstance(b, LoopRegion):
            yield from walk_blocks(b.body, path + (b.label,))
        elif isinstance(b, Conditional):
            yield from walk_blocks(b.then_body, path + (b.label, "then"))
            yield from walk_blocks(b.else_body, path + (b.label, "else"))


def schedule(df: Dataflow) -> list:
    """Deterministic topological order of node ids. Same rule as the
    reference (ir.py:253-306): dataflow edges, plus consecutive access
    instances of one array ordered write-after-read / write-after-write;
    ties broken by node-list position."""
    ids = [n.id for n in df.nodes]
    pos = {nid: i for i, nid in enumerate(ids)}
    succ = {nid: set() for nid in ids}
    indeg = dict.fromkeys(ids, 0)
    srcs_of = {}
    dsts_of = {}
    for e in df.edges:
        srcs_of.setdefault(e.dst, []).append(e.src)
        dsts_of.setdefault(e.src, []).append(e.dst)

    def arc(a, b):
        if a != b and b not in succ[a]:
            succ[a].add(b)
            indeg[b] += 1

    for e in df.edges:
        arc(e.src, e.dst)
    chains = {}
    for n in df.nodes:
        if isinstance(n, AccessNode):
            chains.setdefault(n.data, []).append(n.id)
    for chain in chains.values():
        for a, b in zip(chain, chain[1:]):
            writers = srcs_of.get(b, [])
            arc(a, b)
            for reader in dsts_of.get(a, []):
                for w in writers:
                    arc(reader, w)
            for w in writers:
                arc(a, w)
    heap = [pos[n] for n in ids if indeg[n] == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        nid = ids[heapq.heappop(heap)]
        order.append(nid)
        for m in succ[nid]:
            indeg[m] -= 1
            if indeg[m] == 0:
                heapq.heappush(heap, pos[m])
    if len(order) != len(ids):
        raise ValueError("cycle in state dataflow graph")
    return order


def number_writes(program: Program):
    """Static write versions in program order (reference versions.py:88-105):
    returns ({(state label, access id): version}, {(data, version): loop labels})."""
    counter = dict.fromkeys(program.descriptors, 0)
    version_of = {}
    loops_of = {}

    def region(blocks, loops):
        for b in blocks:
            if isinstance(b, State):
                written = {e.dst for e in b.graph.edges}
                for n in b.graph.nodes:
                    if isinstance(n, AccessNode) and n.id in written:
                        counter[n.data] = counter.get(n.data, 0) + 1
                        v = counter[n.data]
                        version_of[(b.label, n.id)] = v
                        loops_of[(n.data, v)] = loops
            elif isinstance(b, LoopRegion):
                region(b.body, loops + (b.label,))
            elif isinstance(b, Conditional):
                region(b.then_body, loops)
                region(b.else_body, loops)

    region(program.region, ())
    return version_of, loops_of


def pristine_inputs(program: Program) -> set:
    written = set()
    for _, b in walk_blocks(program.region):
        if isinstance(b, State):
            access = {n.id for n in b.graph.nodes if isinstance(n, AccessNode)}
            written |= {e.data for e in b.graph.edges if e.dst in access}
    return {d.name for d in program.descriptors.values() if d.role == "input" and d.name not in written}


# ---------------------------------------------------------------------------
# structural adoption of reference objects


def _adopt_expr(e):
    cls = type(e).__name__
    if isinstance(e, (Const, Name, Unary, Binary, Index)):
        return e
    if cls == "Const":
        return Const(e.value)
    if cls == "Name":
        return Name(e.id)
    if cls == "Unary":
        return Unary(e.op, _adopt_expr(e.x))
    if cls == "Binary":
        return Binary(e.op, _adopt_expr(e.x), _adopt_expr(e.y))
    if cls == "Index":
        return Index(e.base, tuple(_adopt_expr(i) for i in e.indices))
    raise TypeError(f"cannot adopt expression {e!r}")


def _adopt_df(df) -> Dataflow:
    out = Dataflow()
    for n in df.nodes:
        cls = type(n).__name__
        if cls == "AccessNode":
            out.nodes.append(AccessNode(n.id, n.data))
        elif cls == "Tasklet":
            out.nodes.append(Tasklet(n.id, tuple(n.ins), tuple(n.outs),
                                     {k: _adopt_expr(v) for k, v in n.body.items()}, n.group))
        elif cls == "LibraryNode":
            out.nodes.append(LibraryNode(n.id, n.kind, n.op, n.const, bool(n.ta), bool(n.tb), n.group))
        elif cls == "MapNode":
            out.nodes.append(MapNode(n.id, tuple(n.params),
                                     tuple(tuple(_adopt_expr(p) for p in r) for r in n.ranges),
                                     _adopt_df(n.body), n.group))
        else:
            raise TypeError(f"cannot adopt node {n!r}")
    for e in df.edges:
        out.edges.append(Memlet(e.src, e.src_conn, e.dst, e.dst_conn, e.data,
                                None if e.subset is None else tuple(_adopt_expr(s) for s in e.subset),
                                e.wcr))
    return out


def _adopt_region(region) -> list:
    out = []
    for b in region:
        cls = type(b).__name__
        if cls == "State":
            out.append(State(b.label, _adopt_df(b.graph)))
        elif cls == "LoopRegion":
            out.append(LoopRegion(
                b.label, b.iterator, _adopt_expr(b.init), _adopt_expr(b.bound), b.cmp,
                _adopt_expr(b.update), _adopt_region(b.body),
                None if b.inverse is None else _adopt_expr(b.inverse),
                bool(b.reversed_simulate), b.replay_of, b.reverse_of,
            ))
        elif cls == "Conditional":
            out.append(Conditional(b.label, _adopt_expr(b.condition), _adopt_region(b.then_body),
                                   _adopt_region(b.else_body), b.trace_ref))
        else:
            raise TypeError(f"cannot adopt block {b!r}")
    return out


def adopt(program) -> Program:
    """Return ``program`` as this module's ``Program`` (identity for ours;
    structural copy of a reference gradflow ``Program``)."""
    if isinstance(program, Program):
        return program
    descs = {
        k: DataDescriptor(d.name, d.element_kind, tuple(_adopt_expr(s) for s in d.shape), d.role)
        for k, d in program.descriptors.items()
    }
    return Program(descs, tuple(program.parameters), _adopt_region(program.region),
                   program.dependent, tuple(program.independents))


def adopt_forwarding(forwarding) -> dict:
    out = {}
    for name, e in (forwarding or {}).items():
        cands = tuple(Candidate(c.version, tuple(tuple(d) for d in c.directives)) for c in e.candidates)
        out[name] = ForwardingEntry(e.name, e.data, cands)
    return out


# ---------------------------------------------------------------------------
# JSON wire format (format_version 1)

FORMAT_VERSION = 1


def _ex(s, where):
    if not isinstance(s, str):
        raise ProgramSyntaxError(f"expected expression string at {where}")
    return parse_sexpr(s)


def _df_from(doc, where) -> Dataflow:
    df = Dataflow()
    for i, n in enumerate(doc.get("nodes", [])):
        t = n.get("type")
        w = f"{where}/nodes/{i}"
        if t == "access":
            df.nodes.append(AccessNode(n["id"], n["data"]))
        elif t == "tasklet":
            df.nodes.append(Tasklet(n["id"], tuple(n["ins"]), tuple(n["outs"]),
                                    {k: _ex(v, w) for k, v in n["body"].items()}, n.get("group")))
        elif t in ("matmul", "reduce_sum", "ew_unary", "ew_binary"):
            const = n.get("const")
            df.nodes.append(LibraryNode(n["id"], t, n.get("op"), None if const is None else float(const),
                                        bool(n.get("ta", False)), bool(n.get("tb", False)), n.get("group")))
        elif t == "map":
            df.nodes.append(MapNode(n["id"], tuple(n["params"]),
                                    tuple(tuple(_ex(p, w) for p in r) for r in n["ranges"]),
                                    _df_from(n, w), n.get("group")))
        else:
            raise ProgramSyntaxError(f"unknown node type '{t}' at {w}")
    for i, e in enumerate(doc.get("edges", [])):
        sub = e.get("subset")
        df.edges.append(Memlet(e["src"], e.get("src_conn"), e["dst"], e.get("dst_conn"), e["data"],
                               None if sub is None else tuple(_ex(s, f"{where}/edges/{i}") for s in sub),
                               e.get("wcr")))
    return df


def _region_from(blocks, where) -> list:
    out = []
    for i, b in enumerate(blocks):
        w = f"{where}/{i}"
        k = b.get("kind")
        if k == "state":
            out.append(State(b["label"], _df_from(b, w)))
        elif k == "loop":
            rev = b.get("reversal")
            out.append(LoopRegion(
                b["label"], b["iterator"], _ex(b["init"], w), _ex(b["bound"], w), b["cmp"],
                _ex(b["update"], w), _region_from(b["body"], w + "/body"),
                None if b.get("inverse") is None else _ex(b["inverse"], w),
                rev == "simulate", rev.get("replay_of") if isinstance(rev, dict) else None,
                b.get("reverse_of"),
            ))
        elif k == "branch":
            out.append(Conditional(b["label"], _ex(b["condition"], w), _region_from(b["then"], w + "/then"),
                                   _region_from(b["else"], w + "/else"), b.get("trace_ref")))
        elif k == "while":
            raise UnsupportedLoop("while loops have no statically analyzable iteration space")
        else:
            raise ProgramSyntaxError(f"unknown block kind '{k}' at {w}")
    return out


def program_from_dict(doc: dict) -> Program:
    if doc.get("format_version") != FORMAT_VERSION:
        raise ProgramSyntaxError(f"unsupported format version {doc.get('format_version')}")
    descs = {}
    for d in doc["descriptors"]:
        descs[d["name"]] = DataDescriptor(d["name"], d["element_kind"],
                                          tuple(_ex(s, "descriptors") for s in d["shape"]), d["role"])
    return Program(descs, tuple(doc["parameters"]), _region_from(doc["region"], "region"),
                   doc["dependent"], tuple(doc["independents"]))


def load_program(text_or_path) -> Program:
    text = text_or_path
    if not str(text_or_path).lstrip().startswith("{"):
        with open(text_or_path) as f:
            text = f.read()
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ProgramSyntaxError(f"not valid JSON: {exc}") from None
    return program_from_dict(doc)


def _df_to(df: Dataflow) -> dict:
    nodes = []
    for n in df.nodes:
        if isinstance(n, AccessNode):
            nodes.append({"id": n.id, "type": "access", "data": n.data})
        elif isinstance(n, Tasklet):
            d = {"id": n.id, "type": "tasklet", "ins": list(n.ins), "outs": list(n.outs),
                 "body": {k: to_sexpr(v) for k, v in n.body.items()}}
            if n.group is not None:
                d["group"] = n.group
            nodes.append(d)
        elif isinstance(n, LibraryNode):
            d = {"id": n.id, "type": n.kind}
            if n.kind == "matmul":
                d.update(ta=n.ta, tb=n.tb)
            if n.kind in ("ew_unary", "ew_binary"):
                d["op"] = n.op
            if n.kind == "ew_unary" and n.const is not None:
                d["const"] = n.const
            if n.group is not None:
                d["group"] = n.group
            nodes.append(d)
        else:
            d = {"id": n.id, "type": "map", "params": list(n.params),
                 "ranges": [[to_sexpr(a) for a in r] for r in n.ranges]}
            d.update(_df_to(n.body))
            if n.group is not None:
                d["group"] = n.group
            nodes.append(d)
    edges = []
    for e in df.edges:
        d = {"src": e.src, "dst": e.dst, "data": e.data}
        if e.src_conn is not None:
            d["src_conn"] = e.src_conn
        if e.dst_conn is not None:
            d["dst_conn"] = e.dst_conn
        if e.subset is not None:
            d["subset"] = [to_sexpr(s) for s in e.subset]
        if e.wcr is not None:
            d["wcr"] = e.wcr
        edges.append(d)
    return {"nodes": nodes, "edges": edges}


def _region_to(region) -> list:
    out = []
    for b in region:
        if isinstance(b, State):
            d = {"kind": "state", "label": b.label}
            d.update(_df_to(b.graph))
        elif isinstance(b, LoopRegion):
            d = {"kind": "loop", "label": b.label, "iterator": b.iterator, "init": to_sexpr(b.init),
                 "bound": to_sexpr(b.bound), "cmp": b.cmp, "update": to_sexpr(b.update),
                 "body": _region_to(b.body)}
            if b.inverse is not None:
                d["inverse"] = to_sexpr(b.inverse)
            if b.reversed_simulate:
                d["reversal"] = "simulate"
            elif b.replay_of is not None:
                d["reversal"] = {"replay_of": b.replay_of}
            if b.reverse_of is not None:
                d["reverse_of"] = b.reverse_of
        else:
            d = {"kind": "branch", "label": b.label, "condition": to_sexpr(b.condition),
                 "then": _region_to(b.then_body), "else": _region_to(b.else_body)}
            if b.trace_ref is not None:
                d["trace_ref"] = b.trace_ref
        out.append(d)
    return out


def program_to_dict(p: Program) -> dict:
    return {
        "format_version": FORMAT_VERSION,
        "parameters": list(p.parameters),
        "descriptors": [{"name": d.name, "element_kind": d.element_kind,
                         "shape": [to_sexpr(s) for s in d.shape], "role": d.role}
                        for d in p.descriptors.values()],
        "dependent": p.dependent,
        "independents": list(p.independents),
        "region": _region_to(p.region),
    }


def dump_program(p: Program) -> str:
    return json.dumps(program_to_dict(p), sort_keys=True, indent=2) + "\n"


def forwarding_from_manifest(doc: dict) -> tuple:
    """Read the reference ``gradflow diff`` manifest (cli.py:223-237):
    returns (forwarding dict, required set)."""
    fw = {}
    for e in doc.get("entries", []):
        cands = tuple(Candidate(int(c["version"]), tuple(tuple(d) for d in c["directives"]))
                      for c in e["candidates"])
        fw[e["name"]] = ForwardingEntry(e["name"], e["data"], cands)
    required = frozenset((d, int(v)) for d, v in doc.get("required", []))
    return fw, required


def manifest_from_forwarding(forwarding: dict, required) -> dict:
    return {
        "required": sorted([d, v] for d, v in required),
        "entries": [
            {"name": e.name, "data": e.data,
             "candidates": [{"version": c.version, "directives": [list(d) for d in c.directives]}
                            for c in e.candidates]}
            for e in sorted(forwarding.values(), key=lambda e: e.name)
        ],
    }
