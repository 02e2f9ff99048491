"""Reference-facing entry points, executed on the B200 engine.

Mirrors the reference signatures so the engine is a drop-in for the hot
path:

* ``gradient(program, inputs, params=None, *, seed=1.0, trip_limit=None,
  bundle=None) -> GradientResult`` (reference autodiff.py:1153-1184)
* ``run_planned(result, inputs, params=None, *, seed=1.0, trip_limit=None)``
  (reference checkpointing.py:903-957)
* ``run_forward`` / ``run_backward`` (reference interpreter.py:621-695), the
  executor-level seam.
* ``plan(program, limit_mib, params=None, *, trip_limit=None)``: the ILP
  planner is host code and stays the reference's own (checkpointing.py:
  863-900); this wrapper calls it when the reference is installed.

The AD transform (``build_backward``) and the planner are host-side and run
once per (program, params, budget); on a machine without the reference they
arrive as the reference's own serialized artifacts (``load_bundle``,
``load_plan``: the ``gradflow diff`` / ``gradflow plan --emit`` files).
Everything on the data path runs as CUDA launches; there is no CPU
execution path.
"""
from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass, field

import numpy as np

from .errors import EngineError, ShapeMismatch, UnboundName, UnsupportedConstruct
from .ir import (
    Program,
    adopt,
    adopt_forwarding,
    dump_program,
    eval_int,
    forwarding_from_manifest,
    load_program,
    manifest_from_forwarding,
    number_writes,
    pristine_inputs,
)
from .lowering import Lowering, LTape, NeedValues, ProgramRun, required_record
from .runtime import NP_DTYPE, Executable, HostEnv

# ---------------------------------------------------------------------------
# bundles (what the host AD / planner hands to the engine)


@dataclass
class Bundle:
    """Engine view of the reference ``BackwardBundle`` (autodiff.py:428-436)."""

    backward: Program
    forwarding: dict
    required: frozenset


@dataclass
class PlanBundle:
    """Engine view of a reference ``PlanResult`` (checkpointing.py:852-860):
    the rewritten forward/backward pair plus what ``run_planned`` derives
    from it (record set, forwarding subset, names of kept copies)."""

    forward: Program
    backward: Program
    keep: frozenset
    forwarding: dict
    stored: tuple
    report: dict = field(default_factory=dict)


@dataclass
class RunResult:
    env: dict
    value: object
    op_count: int
    tape: object = None


@dataclass
class GradientResult:
    value: object
    grads: dict
    forward: object
    backward: object
    bundle: object


def fused_backward(plan: "PlanBundle") -> Program:
    """The plan's reverse program with its elementwise recompute stages
    evaluated inside the consuming adjoint kernels (recompute.py; the
    north_star's "recomputation fused into the adjoint kernel that consumes
    it"). GFB_FUSE_RECOMPUTE=0 runs the reference's rec_* blocks as written."""
    if os.environ.get("GFB_FUSE_RECOMPUTE", "1") == "0":
        return plan.backward
    got = plan.__dict__.get("_fused")
    if got is None or got[0] is not plan.backward:
        from .recompute import fuse_recompute

        prog, names = fuse_recompute(plan.backward)
        got = plan.__dict__["_fused"] = (plan.backward, prog, tuple(names))
    return got[1]


def _ref_available() -> bool:
    import importlib.util

    return importlib.util.find_spec("gradflow") is not None


def as_bundle(bundle) -> Bundle:
    if isinstance(bundle, Bundle):
        return bundle
    return Bundle(adopt(bundle.backward), adopt_forwarding(bundle.forwarding), frozenset(bundle.required))


def host_build_backward(program) -> Bundle:
    """Run the reference AD transform on the host (it is not on the data
    path). Needs the reference package; otherwise pass ``bundle=``."""
    if not _ref_available():
        raise UnsupportedConstruct(
            "build_backward is the reference's host-side AD transform and the reference is not installed "
            "here: pass bundle=load_bundle(<prog>.bwd.json, <prog>.fwdreq.json)")
    from gradflow.autodiff import build_backward  # type: ignore
    from gradflow.frontend import parse_program  # type: ignore

    ref_prog = program if not isinstance(program, Program) else parse_program(dump_program(program))
    return as_bundle(build_backward(ref_prog))


def load_bundle(bwd_path: str, manifest_path: str) -> Bundle:
    with open(manifest_path) as f:
        fw, required = forwarding_from_manifest(json.load(f))
    return Bundle(load_program(bwd_path), fw, required)


def save_bundle(bundle: Bundle, stem: str):
    with open(stem + ".bwd.json", "w") as f:
        f.write(dump_program(bundle.backward))
    with open(stem + ".fwdreq.json", "w") as f:
        json.dump(manifest_from_forwarding(bundle.forwarding, bundle.required), f, indent=2)


def as_plan(result) -> PlanBundle:
    if isinstance(result, PlanBundle):
        return result
    # reference PlanResult -> the sets run_planned derives (checkpointing.py:917-942)
    fwd = adopt(result.forward)
    bwd = adopt(result.backward)
    fw_all = adopt_forwarding(result.bundle.forwarding)
    keep = {(fv.data, v) for fv in result.fvs if fv.forced for v in fv.versions}
    forwarding = {}
    for name, e in fw_all.items():
        if len(fwd.descriptors[e.data].shape) == 0:
            forwarding[name] = e
            keep |= {(e.data, c.version) for c in e.candidates}
    for fv in result.fvs:
        if fv.forced:
            forwarding[fv.name] = fw_all[fv.name]
    stored = tuple(fv.name for fv, v in zip(result.fvs, result.solution.assignment) if v and not fv.forced)
    return PlanBundle(fwd, bwd, frozenset(keep), forwarding, stored, dict(result.report))


def save_plan(plan: PlanBundle, stem: str):
    with open(stem + ".fwd.json", "w") as f:
        f.write(dump_program(plan.forward))
    with open(stem + ".bwd.json", "w") as f:
        f.write(dump_program(plan.backward))
    doc = {
        "keep": sorted([d, v] for d, v in plan.keep),
        "stored": list(plan.stored),
        "forwarding": manifest_from_forwarding(plan.forwarding, frozenset())["entries"],
        "report": plan.report,
    }
    with open(stem + ".plan.json", "w") as f:
        json.dump(doc, f, indent=2, default=str)


def plan_from_reference_artifacts(emit_stem: str, report, manifest_path: str) -> PlanBundle:
    """A plan from what the reference CLI emits, without the reference:
    ``gradflow plan PROG --emit STEM --json`` writes the rewritten
    ``STEM.fwd.json`` / ``STEM.bwd.json`` (cli.py:251-253) and prints the
    report (checkpointing.py:879-899); ``gradflow diff PROG`` writes the
    forwarding manifest (cli.py:223-237). ``run_planned``'s record set,
    forwarding subset and stored copies (checkpointing.py:917-942) follow
    from those: a forwarded value's versions are its manifest candidates'
    (collect_forwarded, checkpointing.py:255), scalars always ride the tape,
    forced values are recorded, and unforced ``store`` decisions travel by
    name. ``report`` is the parsed JSON or a path to it."""
    if isinstance(report, str):
        with open(report) as f:
            report = json.load(f)
    fwd = load_program(emit_stem + ".fwd.json")
    bwd = load_program(emit_stem + ".bwd.json")
    with open(manifest_path) as f:
        fw_all, _ = forwarding_from_manifest(json.load(f))
    keep, forwarding, stored = set(), {}, []
    for name, e in fw_all.items():
        if len(fwd.descriptors[e.data].shape) == 0:
            forwarding[name] = e
            keep |= {(e.data, c.version) for c in e.candidates}
    for v in report["values"]:
        e = fw_all.get(v["name"])
        if e is None:
            raise UnboundName(f"plan report names '{v['name']}', which the forwarding manifest does not hold")
        if v["forced"]:
            forwarding[v["name"]] = e
            keep |= {(e.data, c.version) for c in e.candidates}
        elif v["decision"] == "store":
            stored.append(v["name"])
    return PlanBundle(fwd, bwd, frozenset(keep), forwarding, tuple(stored), dict(report))


def load_plan(stem: str, manifest: str | None = None) -> PlanBundle:
    """``stem.plan.json`` (``save_plan``), or, given the ``gradflow diff``
    manifest, the reference CLI's own ``stem.report.json`` next to its
    ``--emit`` programs (``plan_from_reference_artifacts``)."""
    if not os.path.exists(stem + ".plan.json") and manifest is not None:
        return plan_from_reference_artifacts(stem, stem + ".report.json", manifest)
    with open(stem + ".plan.json") as f:
        doc = json.load(f)
    fw, _ = forwarding_from_manifest({"entries": doc["forwarding"]})
    return PlanBundle(load_program(stem + ".fwd.json"), load_program(stem + ".bwd.json"),
                      frozenset((d, int(v)) for d, v in doc["keep"]), fw, tuple(doc["stored"]),
                      doc.get("report", {}))


# ---------------------------------------------------------------------------
# executable construction


def _check_inputs(program: Program, inputs: dict, params: dict, *, batch=()):
    """Declared shapes of the inputs (reference _prepare_inputs,
    interpreter.py:604-618). An input may carry the leading ``batch`` dims
    (``batch_of``); any other leading dims are rejected."""
    shapes = {}
    for name, value in inputs.items():
        desc = program.descriptors.get(name)
        if desc is None:
            raise UnboundName(f"input '{name}' is not declared")
        declared = tuple(eval_int(d, params) for d in desc.shape)
        shape = tuple(getattr(value, "shape", np.shape(value)))
        if desc.shape and tuple(shape[len(shape) - len(declared):]) != declared:
            raise ShapeMismatch(f"input '{name}': trailing shape {shape} does not end with {declared}")
        if len(shape) != len(declared) and tuple(shape[:len(shape) - len(declared)]) != tuple(batch):
            raise ShapeMismatch(f"input '{name}': leading dims {shape[:len(shape) - len(declared)]} are not the "
                                f"batch shape {tuple(batch)}")
        shapes[name] = declared
    return shapes


def batch_of(program: Program, inputs: dict) -> tuple:
    """The leading batch shape (reference Executor._batch_shape,
    interpreter.py:161-169): the extra leading dims of the first input that
    has any; inputs without them are shared by every batch element."""
    for name, value in inputs.items():
        desc = program.descriptors.get(name)
        if desc is None:
            continue
        shape = tuple(getattr(value, "shape", np.shape(value)))
        if len(shape) > desc.rank:
            return shape[:len(shape) - desc.rank]
    return ()


def _element(program: Program, inputs: dict, batch: tuple, idx: tuple) -> dict:
    """Inputs of one batch element (batched arrays indexed, shared ones as is)."""
    out = {}
    for name, value in inputs.items():
        desc = program.descriptors[name]
        nd = len(getattr(value, "shape", np.shape(value)))
        out[name] = value[idx] if nd > desc.rank else value
    return out


def _batched(program: Program, inputs: dict, batch: tuple, run_one, keys):
    """Run ``run_one(element_inputs, first)`` for every batch element in order;
    each call returns {key: array}; results are stacked to batch + shape.
    Batch elements are independent in the reference (every operation acts
    per element along the leading dims; control flow must agree across the
    batch, else BatchDivergence, interpreter.py:190-196), so element-wise
    execution of the same launch list is the same computation. Device inputs
    are uploaded once; element copies are device-to-device."""
    import torch

    dev_inputs = {}
    for k, v in inputs.items():
        desc = program.descriptors[k]
        if len(np.shape(v)) > desc.rank and not isinstance(v, torch.Tensor) and torch.cuda.is_available():
            dev_inputs[k] = torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=NP_DTYPE[desc.element_kind]))
                                             ).cuda()
        else:
            dev_inputs[k] = v
    results = {}
    first = True
    for idx in np.ndindex(*batch):
        got = run_one(_element(program, dev_inputs, batch, idx), first)
        for k in keys:
            v = got.get(k)
            if v is None:
                continue
            if k not in results:
                results[k] = np.empty(tuple(batch) + np.shape(v), dtype=np.asarray(v).dtype)
            results[k][idx] = v
        first = False
    return results


def _init_env(low: Lowering, program: Program, shapes: dict, prefix: str):
    env, inputs = {}, {}
    for name, shape in shapes.items():
        desc = program.descriptors[name]
        b = low.new_buffer(prefix + name, shape, desc.element_kind, fresh=False)
        env[name] = b
        inputs[name] = b
    return env, inputs


@dataclass
class Lowered:
    low: Lowering
    inputs: dict
    outputs: dict
    seed_buf: object
    forward_env: dict
    backward_env: dict
    tape: LTape
    forward_program: Program
    backward_program: Program


class NeedsInputs(UnsupportedConstruct):
    """Lowering reached data-dependent control flow without input values."""


def probe_values(nv: NeedValues, inputs: dict, seed=1.0) -> dict:
    """Run the launches lowered before a data-dependent decision and read the
    snapshots it needs (host copies, name -> ndarray)."""
    low = nv.low
    slots = list(nv.slots.values())
    low.finish(slots)
    exe = Executable(low, low.entry_inputs, {}, seed_buf=low.entry_seed, use_graph=False,
                     pinned=[low.resolve(b) for b in slots])
    exe.run({k: inputs[k] for k in low.entry_inputs}, seed)
    return {n: exe.view(low.resolve(b)).cpu().numpy().copy() for n, b in nv.slots.items()}


class _Known(list):
    """Decision values known before lowering, plus the incremental prober
    the Lowering calls for the ones met while lowering."""

    def __init__(self, probe=None):
        super().__init__()
        self.probe = probe


def probe_lower(lower, inputs: dict | None, seed=1.0):
    """``lower(known)`` with the data-dependent decisions (reference branches
    / loop headers, interpreter.py:210-219, 342-347, evaluated at the same
    program point) resolved as they are met: a ``ProbeRuntime`` runs the
    launches emitted since the previous decision and reads its snapshots,
    so the lowering runs once. Without inputs, or on a box without a GPU,
    each ``NeedValues`` ends the attempt and the prefix is probed from
    scratch (``probe_values``)."""
    from .runtime import ProbeRuntime

    prober = None
    if inputs is not None:
        try:
            prober = ProbeRuntime(inputs, seed)
        except EngineError:
            prober = None
    known = _Known(prober)
    while True:
        try:
            return lower(known)
        except NeedValues as nv:
            if inputs is None:
                raise NeedsInputs(
                    f"control flow depends on runtime data ({', '.join(sorted(nv.slots))}); "
                    "the launch list needs input values to be lowered") from None
            known.append(probe_values(nv, inputs, seed))


def lower_gradient(program: Program, bundle: Bundle, params: dict, shapes: dict, *, trip_limit=None,
                   record=None, plan: PlanBundle | None = None, fuse_small=False, known=None) -> Lowered:
    """Forward (recording the tape) + backward as one launch list."""
    low = Lowering(trip_limit=trip_limit, fuse_small=fuse_small, known=known)
    fwd_prog = plan.forward if plan else program
    bwd_prog = fused_backward(plan) if plan else bundle.backward
    forwarding = plan.forwarding if plan else bundle.forwarding
    rec = set(plan.keep) if plan else set(bundle.required if record is None else record)
    fenv, inputs = _init_env(low, fwd_prog, shapes, "")
    low.entry_inputs = inputs
    tape = LTape()
    for name, b in list(fenv.items()):
        if (name, 0) in rec:
            slot = low.new_buffer(f"{name}@v0", b.shape, b.kind, fresh=False)
            from .lowering import CopyOp

            low.emit(CopyOp(slot, b))
            tape.values[(name, 0, ())] = slot
    fr = ProgramRun(low, fwd_prog, params, fenv, record=rec, tape=tape, versions=number_writes(fwd_prog))
    fr.run()
    dep = fenv.get(fwd_prog.dependent)
    if dep is None:
        raise UnboundName(f"dependent '{fwd_prog.dependent}' was never written")
    # backward env: pristine caller inputs alias the forward's input buffers
    benv = {}
    for name in bwd_prog.descriptors:
        if name in inputs and name in pristine_inputs(fwd_prog):
            benv[name] = inputs[name]
    if plan:
        for name in plan.stored:
            if name in bwd_prog.descriptors:
                if name not in fenv:
                    raise UnboundName(f"planned copy '{name}' was never written by the forward program")
                benv[name] = fenv[name]
    seed_name = fwd_prog.dependent + "__grad"
    seed_buf = None
    if seed_name in bwd_prog.descriptors and seed_name not in benv:
        seed_buf = low.new_buffer(seed_name, (), bwd_prog.descriptors[seed_name].element_kind, fresh=False)
        benv[seed_name] = seed_buf
    low.entry_seed = seed_buf
    br = ProgramRun(low, bwd_prog, params, benv, src_tape=tape, forwarding=forwarding)
    br.run()
    outputs = {"value": dep}
    for ind in fwd_prog.independents:
        g = benv.get(ind + "__grad")
        if g is not None:
            outputs["grad:" + ind] = g
    low.finish(list(outputs.values()))
    outputs = {k: low.resolve(b) for k, b in outputs.items()}
    fenv = {k: low.resolve(b) for k, b in fenv.items()}
    benv = {k: low.resolve(b) for k, b in benv.items()}
    return Lowered(low, inputs, outputs, seed_buf, fenv, benv, tape, fwd_prog, bwd_prog)


def build_gradient_executable(program: Program, bundle: Bundle, params: dict, shapes: dict, *, trip_limit=None,
                              record=None, plan: PlanBundle | None = None, inputs: dict | None = None,
                              seed=1.0, pin_env=False) -> Executable:
    """``inputs`` (host or device values) are needed only by programs whose
    control flow reads runtime data; the launch list then holds the path
    those inputs take (``Executable.decisions_hold`` re-checks it).
    ``pin_env`` keeps every named array of the forward and reverse runs out
    of the recycling arena, so ``RunResult.env`` holds all of them like the
    reference's (interpreter.py:78-83); planned runs leave it off, since
    their device peak is bounded by the plan's budget."""
    lw = probe_lower(lambda known: lower_gradient(program, bundle, params, shapes, trip_limit=trip_limit,
                                                  record=record, plan=plan, known=known), inputs, seed)
    pinned = [b for b in list(lw.forward_env.values()) + list(lw.backward_env.values())] if pin_env else []
    exe = Executable(lw.low, lw.inputs, lw.outputs, seed_buf=lw.seed_buf, pinned=pinned)
    exe.forward_env, exe.backward_env, exe.tape = lw.forward_env, lw.backward_env, lw.tape
    exe.forward_program, exe.backward_program = lw.forward_program, lw.backward_program
    return exe


# executable cache: (content fingerprints of the programs, params, shapes)
# -> Executable. Keys are structural, so a program mutated in place (e.g.
# ``prog.independents = ...``) or a new object at a recycled address never
# reuses another program's launch list.
_CACHE: dict = {}
_CACHE_MAX = int(os.environ.get("GFB_CACHE", "4"))
# host AD results of ``gradient(bundle=None)`` by forward-program fingerprint;
# kept apart from the executable LRU so they neither evict nor get evicted
_BUNDLES: dict = {}


def fingerprint(prog: Program) -> str:
    """Content hash of a program (its canonical wire-format serialization)."""
    return hashlib.sha1(dump_program(prog).encode()).hexdigest()


def _cached(key, keep_alive, build):
    exe = _CACHE.get(key)
    if exe is None:
        exe = build()
        if len(_CACHE) >= _CACHE_MAX:
            _CACHE.pop(next(iter(_CACHE)))
        _CACHE[key] = exe
        exe._keep_alive = keep_alive
    return exe


def run_checked(exe: Executable, inputs, seed, rebuild, *, sync=True) -> Executable:
    """Run ``exe``; when it was lowered along a data-dependent path, re-check
    the decisions BEFORE reading the device error word. A call whose inputs
    take another arm may have raised a domain error on the stale arm (``if
    x > 0: log(x)`` called with x <= 0), which the reference never evaluates
    (interpreter.py:342-351 decides first): that run is discarded, the
    program is lowered along the new path and run again."""
    if not exe.low.decisions:
        exe.run(inputs, seed, sync=sync)
        return exe
    exe.run(inputs, seed, sync=False)
    if exe.decisions_hold():
        if sync:
            exe.check()
        return exe
    exe = rebuild()
    exe.run(inputs, seed, sync=sync)
    return exe


def _run_guarded(key, keep_alive, build, inputs, seed):
    """Run the cached executable; when its data-dependent decisions do not
    hold for these inputs, lower again along the path they take."""
    exe = _cached(key, keep_alive, build)
    new = run_checked(exe, inputs, seed, build)
    if new is not exe:
        new._keep_alive = keep_alive
        _CACHE[key] = new
    return new


def clear_cache():
    _CACHE.clear()
    _BUNDLES.clear()
    _SLABS.clear()


def _result(exe: Executable, program: Program, inputs: dict, bundle) -> GradientResult:
    value = exe.output_host("value")
    grads = {}
    for ind in program.independents:
        key = "grad:" + ind
        if key in exe.outputs:
            grads[ind] = exe.output_host(key)
        else:
            ref = np.asarray(inputs[ind])
            grads[ind] = np.zeros(ref.shape, dtype=NP_DTYPE[program.descriptors[ind].element_kind])
    # env: host numpy arrays like the reference's, copied on first access
    # (runtime.HostEnv); entries whose HBM the liveness arena recycled (only
    # in planned runs, whose peak is bounded by the budget) are omitted
    kept = getattr(exe, "keep_bids", None)
    fenv = HostEnv(exe, {k: b for k, b in exe.forward_env.items() if kept is None or b.root().bid in kept})
    benv = HostEnv(exe, {k: b for k, b in exe.backward_env.items() if kept is None or b.root().bid in kept})
    fwd = RunResult(env=fenv, value=value, op_count=exe.flops, tape=exe.tape)
    bwd = RunResult(env=benv, value=None, op_count=exe.flops)
    res = GradientResult(value=value, grads=grads, forward=fwd, backward=bwd, bundle=bundle)
    res._decisions = tuple(k for _, _, k in exe.low.decisions)  # the control-flow path taken
    return res


_SLABS: dict = {}


def _slab_gradient(program, prog, fp, inputs, params, seed, trip_limit, bundle, group):
    """``gradient(..., group=pg)``: the stencil program slab-decomposed over
    the ranks of ``pg`` (decomp.py), one GPU per rank. Every rank passes the
    full inputs and gets the value and the full gradients back."""
    from .decomp import SlabEngine

    shapes = _check_inputs(prog, inputs, params)
    key = (fp, None if bundle is None else fingerprint(as_bundle(bundle).backward), tuple(sorted(params.items())),
           tuple(sorted(shapes.items())), trip_limit, id(group))
    eng = _SLABS.get(key)
    if eng is None:
        eng = SlabEngine(prog, bundle if bundle is not None else _BUNDLES.get(fp) or host_build_backward(program),
                         params, group=group, trip_limit=trip_limit)
        eng._keep_alive = (program, bundle, group)
        _SLABS[key] = eng
    return eng.full_gradient(inputs, seed)


def gradient(program, inputs: dict, params: dict | None = None, *, seed=1.0, trip_limit=None, bundle=None,
             group=None):
    """Reference ``gradient`` (autodiff.py:1153) executed on the B200.

    ``group`` (engine extension, keyword-only, default None): a
    torch.distributed process group; the program is then slab-decomposed
    over its ranks (one GPU each, NCCL halo exchange per timestep)."""
    params = dict(params or {})
    prog = adopt(program)
    fp = fingerprint(prog)
    if group is not None:
        return _slab_gradient(program, prog, fp, inputs, params, seed, trip_limit, bundle, group)
    batch = batch_of(prog, inputs)
    if batch:
        return _gradient_batched(program, prog, inputs, params, batch, seed, trip_limit, bundle)
    if bundle is None:
        bundle_eng = _BUNDLES.get(fp)
        if bundle_eng is None:
            bundle_eng = _BUNDLES[fp] = host_build_backward(program)
        bfp = "auto"
    else:
        bundle_eng = as_bundle(bundle)
        bfp = fingerprint(bundle_eng.backward)
    shapes = _check_inputs(prog, inputs, params)
    key = ("grad", fp, bfp, tuple(sorted(params.items())), tuple(sorted(shapes.items())), trip_limit)
    build = lambda: build_gradient_executable(prog, bundle_eng, params, shapes, trip_limit=trip_limit,  # noqa: E731
                                              inputs=inputs, seed=seed, pin_env=True)
    exe = _run_guarded(key, (program, bundle, bundle_eng), build, inputs, seed)
    return _result(exe, prog, inputs, bundle if bundle is not None else bundle_eng)


def _gradient_batched(program, prog, inputs, params, batch, seed, trip_limit, bundle):
    """``gradient`` over leading batch dims: every element through the cached
    launch list (graph replays), results stacked; an element whose data-
    dependent control flow differs from element 0's raises BatchDivergence
    like the reference (interpreter.py:190-219)."""
    from .errors import BatchDivergence

    _check_inputs(prog, inputs, params, batch=batch)
    paths = []

    def one(elem, first):
        r = gradient(program, elem, params, seed=seed, trip_limit=trip_limit, bundle=bundle)
        paths.append(r._decisions)
        if paths[-1] != paths[0]:
            raise BatchDivergence("a data-dependent branch or loop header differs across the batch")
        out = {"value": np.asarray(r.value)}
        out.update({"grad:" + k: np.asarray(v) for k, v in r.grads.items()})
        return out

    res = _batched(prog, inputs, batch, one, ["value"] + ["grad:" + k for k in prog.independents])
    b = as_bundle(bundle) if bundle is not None else _BUNDLES.get(fingerprint(prog))
    return GradientResult(value=res["value"], grads=_backward_batch(prog, b.backward, b.forwarding, inputs, res),
                          forward=None, backward=None, bundle=bundle)


def _backward_batch(prog, backward, forwarding, inputs, res) -> dict:
    """The reference batches the reverse run only when an input it reads
    carries the batch dims or it reads recorded forward values
    (run_backward sizes the seed and zero-initialised gradients from its own
    env, interpreter.py:681-689, :161-169); otherwise the gradient is the
    unbatched one of a single element (a linear program's adjoint does not
    depend on the point)."""
    batched = bool(forwarding) or any(
        k in backward.descriptors and len(np.shape(v)) > prog.descriptors[k].rank for k, v in inputs.items())
    grads = {}
    for k in prog.independents:
        g = res["grad:" + k]
        grads[k] = g if batched else g.reshape((-1,) + g.shape[g.ndim - prog.descriptors[k].rank:])[0]
    return grads


def run_planned(result, inputs: dict, params: dict | None = None, *, seed=1.0, trip_limit=None):
    """Reference ``run_planned`` (checkpointing.py:903) executed on the B200."""
    params = dict(params or {})
    pb = as_plan(result)
    batch = batch_of(pb.forward, inputs)
    if batch:
        from .errors import BatchDivergence

        _check_inputs(pb.forward, inputs, params, batch=batch)
        paths = []

        def one(elem, first):
            r = run_planned(result, elem, params, seed=seed, trip_limit=trip_limit)
            paths.append(r._decisions)
            if paths[-1] != paths[0]:
                raise BatchDivergence("a data-dependent branch or loop header differs across the batch")
            return {"value": np.asarray(r.value), **{"grad:" + k: np.asarray(v) for k, v in r.grads.items()}}

        res = _batched(pb.forward, inputs, batch, one, ["value"] + ["grad:" + k for k in pb.forward.independents])
        return GradientResult(value=res["value"],
                              grads=_backward_batch(pb.forward, pb.backward, pb.forwarding, inputs, res),
                              forward=None, backward=None, bundle=getattr(result, "bundle", None))
    shapes = _check_inputs(pb.forward, inputs, params)
    key = ("plan", fingerprint(pb.forward), fingerprint(pb.backward), tuple(sorted(pb.keep)), tuple(pb.stored),
           tuple(sorted(params.items())), tuple(sorted(shapes.items())), trip_limit)
    build = lambda: build_gradient_executable(pb.forward, None, params, shapes, trip_limit=trip_limit,  # noqa: E731
                                              plan=pb, inputs=inputs, seed=seed)
    exe = _run_guarded(key, (result,), build, inputs, seed)
    return _result(exe, pb.forward, inputs, getattr(result, "bundle", None))


def plan(program, limit_mib, params=None, *, trip_limit=None):
    """The reference's host-side ILP planner (checkpointing.py:863); its
    result runs on the engine through ``run_planned``."""
    if not _ref_available():
        raise UnsupportedConstruct("plan() is the reference's host ILP planner; load an emitted plan with load_plan()")
    from gradflow.checkpointing import plan as ref_plan  # type: ignore
    from gradflow.frontend import parse_program  # type: ignore

    ref_prog = program if not isinstance(program, Program) else parse_program(dump_program(program))
    return ref_plan(ref_prog, limit_mib, params, trip_limit=trip_limit)


def _forward_batched(prog, inputs, params, batch, trip_limit):
    """``run_forward`` over leading batch dims, record None (the reference FD
    oracle's use, verification.py:96-108): the forward launch list is built
    once and replayed per element as a CUDA graph with device-to-device input
    copies; the dependent of every element lands in a device vector and the
    host synchronises once. Programs with data-dependent control flow run
    element by element and raise BatchDivergence when the path differs."""
    import torch

    from .errors import BatchDivergence

    shapes = _check_inputs(prog, inputs, params, batch=batch)
    key = ("fwd", fingerprint(prog), tuple(sorted(params.items())), tuple(sorted(shapes.items())), trip_limit)

    def build(elem):
        low, env, ins, _tape = probe_lower(lambda known: _lower_forward(prog, shapes, params, None, trip_limit,
                                                                         known), elem)
        dep = env.get(prog.dependent)
        if dep is None:
            raise UnboundName(f"dependent '{prog.dependent}' was never written")
        low.finish([dep])
        return Executable(low, ins, {"value": low.resolve(dep)})

    exe = _CACHE.get(key)
    vals, paths = None, []

    def one(elem, first):
        nonlocal exe, vals
        if exe is None:
            exe = build(elem)
            exe._keep_alive = (prog,)
            _CACHE[key] = exe
        if exe.low.decisions:
            exe = run_checked(exe, elem, 1.0, lambda: build(elem))
            _CACHE[key] = exe
            paths.append(tuple(k for _, _, k in exe.low.decisions))
            if paths[-1] != paths[0]:
                raise BatchDivergence("a data-dependent branch or loop header differs across the batch")
            return {"value": exe.output_host("value")}
        exe.run(elem, sync=False, clear_err=first)
        v = exe.output("value")
        if vals is None:
            vals = torch.empty((int(np.prod(batch)),) + tuple(v.shape), dtype=v.dtype, device=v.device)
        vals[idx_of[0]] = v
        idx_of[0] = idx_of[0] + 1
        return {}

    idx_of = [0]
    res = _batched(prog, inputs, batch, one, ["value"])
    if vals is not None:
        exe.check()
        value = vals.cpu().numpy().reshape(tuple(batch) + tuple(vals.shape[len(batch):]))
    else:
        value = res["value"]
    return RunResult(env={}, value=value, op_count=exe.flops)


def _lower_forward(prog, shapes, params, record, trip_limit, known):
    low = Lowering(trip_limit=trip_limit, known=known)
    env, ins = _init_env(low, prog, shapes, "")
    low.entry_inputs = ins
    tape = LTape() if record is not None else None
    if tape is not None:
        from .lowering import CopyOp

        for name, b in list(env.items()):
            if record == "all" or (name, 0) in record:
                slot = low.new_buffer(f"{name}@v0", b.shape, b.kind, fresh=False)
                low.emit(CopyOp(slot, b))
                tape.values[(name, 0, ())] = slot
    ProgramRun(low, prog, params, env, record=record, tape=tape, versions=number_writes(prog)).run()
    return low, env, ins, tape


def run_forward(program, inputs: dict, params: dict | None = None, *, record=None, trip_limit=None, vinfo=None):
    """Reference ``run_forward`` (interpreter.py:621): the forward program
    alone; ``record`` None, "all" or a set of (name, version). Inputs may
    carry leading batch dims (record None): see ``_forward_batched``."""
    params = dict(params or {})
    prog = adopt(program)
    batch = batch_of(prog, inputs)
    if batch:
        if record is not None:
            raise UnsupportedConstruct("run_forward: recording a tape over a batch is not supported; "
                                       "use gradient() on the batch")
        return _forward_batched(prog, inputs, params, batch, trip_limit)
    shapes = _check_inputs(prog, inputs, params)
    def lower(known):
        low = Lowering(trip_limit=trip_limit, known=known)
        env, ins = _init_env(low, prog, shapes, "")
        low.entry_inputs = ins
        tape = LTape() if record is not None else None
        if tape is not None:
            from .lowering import CopyOp

            for name, b in list(env.items()):
                if record == "all" or (name, 0) in record:
                    slot = low.new_buffer(f"{name}@v0", b.shape, b.kind, fresh=False)
                    low.emit(CopyOp(slot, b))
                    tape.values[(name, 0, ())] = slot
        ProgramRun(low, prog, params, env, record=record, tape=tape, versions=number_writes(prog)).run()
        return low, env, ins, tape

    low, env, ins, tape = probe_lower(lower, inputs)
    dep = env.get(prog.dependent)
    if dep is None:
        raise UnboundName(f"dependent '{prog.dependent}' was never written")
    observed = list(env.values()) + (list(tape.values.values()) if tape else [])
    low.finish(observed)
    exe = Executable(low, ins, {"value": low.resolve(dep)}, use_graph=False,
                     pinned=[low.resolve(b) for b in observed])
    exe.run(inputs)
    out_env = HostEnv(exe, {k: low.resolve(b) for k, b in env.items()})
    res = RunResult(env=out_env, value=exe.output_host("value"), op_count=exe.flops, tape=tape)
    res._exe = exe
    return res


def run_backward(program, backward, inputs: dict, params: dict | None = None, *, tape=None, forwarding=None,
                 seed=1.0, extra_env=None, trip_limit=None):
    """Reference ``run_backward`` (interpreter.py:659). ``tape`` must come
    from this engine's ``run_forward`` (device-resident snapshots)."""
    params = dict(params or {})
    prog = adopt(program)
    bwd = adopt(backward)
    fw = adopt_forwarding(forwarding) if forwarding and not isinstance(next(iter(forwarding.values())), type(None)) \
        else {}
    pass_in = {k: v for k, v in inputs.items() if k in bwd.descriptors}
    extra_in = {k: v for k, v in (extra_env or {}).items() if k in bwd.descriptors}
    seed_name = prog.dependent + "__grad"

    def lower(known):
        low = Lowering(trip_limit=trip_limit, known=known)
        shapes = _check_inputs(bwd, pass_in, params)
        env, ins = _init_env(low, bwd, shapes, "")
        for k, v in extra_in.items():
            b = low.new_buffer(k, tuple(np.shape(v)), bwd.descriptors[k].element_kind, fresh=False)
            env[k] = b
            ins[k] = b
        seed_buf = None
        if seed_name in bwd.descriptors and seed_name not in env:
            seed_buf = low.new_buffer(seed_name, (), bwd.descriptors[seed_name].element_kind, fresh=False)
            env[seed_name] = seed_buf
        low.entry_inputs, low.entry_seed = ins, seed_buf
        ProgramRun(low, bwd, params, env, src_tape=tape, forwarding=fw).run()
        return low, env, ins, seed_buf

    low, env, ins, seed_buf = probe_lower(lower, {**pass_in, **extra_in}, seed)
    low.finish(list(env.values()))
    outputs = {"value": seed_buf} if seed_buf is not None else {}
    exe = Executable(low, ins, outputs, seed_buf=seed_buf, use_graph=False,
                     pinned=[low.resolve(b) for b in env.values()])
    exe.run({**pass_in, **extra_in}, seed)
    out_env = HostEnv(exe, {k: low.resolve(b) for k, b in env.items()})
    return RunResult(env=out_env, value=None if seed_buf is None else exe.output_host("value"), op_count=exe.flops)


class Engine:
    """Device-resident gradient evaluator for one (program, params): the
    object bench.py drives. ``step(device_inputs)`` runs forward+backward on
    inputs already in HBM; ``gradient(host_inputs)`` is the end-to-end call."""

    def __init__(self, program, bundle=None, params=None, shapes=None, *, plan: PlanBundle | None = None,
                 trip_limit=None):
        self.params = dict(params or {})
        self.plan = plan
        self.program = adopt(program) if program is not None else plan.forward
        self.bundle = None if plan else (as_bundle(bundle) if bundle is not None else host_build_backward(program))
        if shapes is None:
            shapes = {n: tuple(eval_int(s, self.params) for s in d.shape)
                      for n, d in self.program.descriptors.items() if d.role == "input"}
        self.shapes = dict(shapes)
        self.trip_limit = trip_limit
        # programs whose control flow reads runtime data are lowered at the
        # first call, along the path its inputs take (api.probe_lower)
        try:
            self.exe = self._build(None)
        except NeedsInputs:
            self.exe = None

    def _build(self, inputs, seed=1.0):
        return build_gradient_executable(self.program, self.bundle, self.params, self.shapes,
                                         trip_limit=self.trip_limit, plan=self.plan, inputs=inputs, seed=seed)

    def _run(self, inputs, seed, sync):
        if self.exe is None:
            self.exe = self._build(inputs, seed)
        self.exe = run_checked(self.exe, inputs, seed, lambda: self._build(inputs, seed), sync=sync)

    def step(self, inputs: dict, seed=1.0, sync=False):
        self._run(inputs, seed, sync)

    def check(self):
        self.exe.check()

    def gradient(self, inputs: dict, seed=1.0) -> GradientResult:
        self._run(inputs, seed, True)
        return _result(self.exe, self.program, inputs, self.bundle)

    def gradients(self, batches, seed=1.0):
        """One ``GradientResult`` per input dict of ``batches``, with host
        inputs in and host results out, pipelined across calls
        (``Executable.run_pipelined``): the next batch's H2D copy and the
        previous result's D2H copy overlap the current batch's launches.
        Results carry value and grads (fresh host arrays); ``forward`` /
        ``backward`` envs are not kept per batch (None). Programs with
        data-dependent control flow run the calls one after another (each
        call's path is known only after its decisions are read back)."""
        if self.exe is None or self.exe.low.decisions:
            for inputs in batches:
                r = self.gradient(inputs, seed)
                yield GradientResult(value=np.array(r.value), grads={k: np.array(v) for k, v in r.grads.items()},
                                     forward=None, backward=None, bundle=self.bundle)
            return
        outs = {k: self.exe.output(k) for k in self.exe.outputs if k == "value" or k.startswith("grad:")}
        for host in self.exe.run_pipelined(batches, outs, seed):
            grads = {}
            for ind in self.program.independents:
                t = host.get("grad:" + ind)
                grads[ind] = t.numpy() if t is not None else np.zeros(
                    self.shapes[ind], dtype=NP_DTYPE[self.program.descriptors[ind].element_kind])
            yield GradientResult(value=host["value"].numpy(), grads=grads, forward=None, backward=None,
                                 bundle=self.bundle)
