"""Host-side (CPU) checks added in round 2: typed errors with the
reference's exception classes, a loop-carried iterator-dependent branch
re-checked after lowering, the reference CLI's plan artifacts consumed
without the reference, and the structural program cache keys."""
import json
import os

import numpy as np
import pytest

import emulator as E
from conftest import GOLD, rel_err, tol_for
from paper_2509_02197_b200 import workloads as W
from paper_2509_02197_b200.api import (
    _check_inputs,
    _init_env,
    fingerprint,
    load_bundle,
    load_plan,
    lower_gradient,
    plan_from_reference_artifacts,
)
from paper_2509_02197_b200.errors import MissingTapeValue, NonTermination, OutOfBounds
from paper_2509_02197_b200.ir import dump_program, load_program
from paper_2509_02197_b200.lowering import Lowering, LTape, NeedValues, ProgramRun

R2 = os.path.join(GOLD, "r2")
R2IDX = json.load(open(os.path.join(R2, "index.json")))
ERRORS = json.load(open(os.path.join(R2, "errors.json")))


def _bundle(name):
    stem = os.path.join(W.PROG_DIR, name)
    return load_program(stem + ".fwd.json"), load_bundle(stem + ".bwd.json", stem + ".fwdreq.json")


def _r2_bundle(name):
    stem = os.path.join(R2, name)
    return load_program(stem + ".fwd.json"), load_bundle(stem + ".bwd.json", stem + ".fwdreq.json")


def _r2_case(cid):
    g = np.load(os.path.join(R2, cid + ".npz"))
    inputs = {k[3:]: g[k] for k in g.files if k.startswith("in:")}
    grads = {k[5:]: g[k] for k in g.files if k.startswith("grad:")}
    return inputs, g["value"], grads


# -- typed errors (reference errors.py; interpreter.py:59-67, :230-233, :511-527)


def test_out_of_bounds_is_typed():
    """A map reaching past the declared extent raises OutOfBounds (reference
    interpreter.py:396-403), statically, before any launch."""
    prog, b = _bundle("jacobi_2d")
    with pytest.raises(OutOfBounds):
        lower_gradient(prog, b, {"N": 6, "TSTEPS": 3}, {"A": (5, 5), "B": (5, 5)})


def test_trip_guard_raises_non_termination_like_the_reference():
    case = ERRORS["trip_limit"]
    assert case["error"] == "NonTermination"
    prog, b = _bundle(case["workload"])
    params = case["params"]
    shapes = {"A": (6, 6), "B": (6, 6)}
    with pytest.raises(NonTermination):
        lower_gradient(prog, b, params, shapes, trip_limit=case["trip_limit"])
    # the guard is "more trips than the limit" (interpreter.py:230): 5 trips pass at limit 5
    lower_gradient(prog, b, params, shapes, trip_limit=params["TSTEPS"] - 1)


@pytest.mark.parametrize("which", ["no_tape", "empty_tape"])
def test_backward_without_recorded_value_raises_missing_tape_value(which):
    case = ERRORS[which]
    assert case["error"] == "MissingTapeValue"
    prog, b = _bundle(case["workload"])
    params = case["params"]
    assert b.forwarding, "atax forwards t"
    low = Lowering()
    env, _ = _init_env(low, b.backward, {"A": (6, 5), "x": (5, 1)}, "")
    env["O__grad"] = low.new_buffer("O__grad", (), "real64", fresh=False)
    tape = None if which == "no_tape" else LTape()
    with pytest.raises(MissingTapeValue):
        ProgramRun(low, b.backward, params, env, src_tape=tape, forwarding=b.forwarding).run()


# -- data-dependent control flow (key functions capture bindings)


def _emulate_probing(prog, bundle, params, inputs):
    shapes = _check_inputs(prog, inputs, params)
    known = []
    while True:
        try:
            lw = lower_gradient(prog, bundle, params, shapes, known=known)
            break
        except NeedValues as nv:
            low = nv.low
            low.finish(list(nv.slots.values()))
            _, pview = E.execute(low, {k: inputs[k] for k in low.entry_inputs}, low.entry_inputs, low.entry_seed)
            known.append({n: np.array(pview(low.resolve(b))) for n, b in nv.slots.items()})
    em, view = E.execute(lw.low, inputs, lw.inputs, lw.seed_buf)
    return lw, em, view


@pytest.mark.parametrize("cid", sorted(c for c in R2IDX["control_flow"] if c.startswith("loop_branch")))
def test_iterator_dependent_branch_matches_reference_and_rechecks(cid):
    """The condition ``(lt t i)`` reads the loop iterator: each of the three
    decisions re-evaluates, after lowering, with the iterator value of its
    own trip (reference interpreter.py:332-351)."""
    prog, b = _r2_bundle("loop_branch")
    inputs, value, grads = _r2_case(cid)
    lw, em, view = _emulate_probing(prog, b, {}, inputs)
    assert rel_err(view(lw.outputs["value"]), value) <= 1e-12
    assert rel_err(view(lw.outputs["grad:t"]), grads["t"]) <= 1e-12
    decisions = lw.low.decisions
    assert len(decisions) == 3
    t = float(inputs["t"])
    for i, (slots, key_fn, key) in enumerate(decisions):
        assert key == (t < i)
        snap = {n: np.array(view(lw.low.resolve(s))) for n, s in slots.items()}
        assert key_fn(snap) == key
        # another t flips exactly the trips whose iterator it crosses
        assert key_fn({"t": np.array(0.5)}) == (0.5 < i)


class _EmuProbe:
    """The api's incremental prober (runtime.ProbeRuntime) on the emulator:
    at each decision it runs only the launches emitted since the previous
    one, on memory it keeps for the whole lowering."""

    def __init__(self, inputs, seed=1.0):
        self.mem = E.Memory()
        self.em = E.Emulator(self.mem)
        self.inputs, self.seed = inputs, seed
        self.done, self.launches, self.calls, self.loaded = 0, 0, 0, False
        self.shims = {}

        class RT:
            pass

        self.rt = RT()
        self.rt.upload = self._upload
        self.rt.workspace_ptr = self.mem.alloc(1 << 16, np.uint8).ctypes.data
        self.rt.err_ptr = self.em.err.ctypes.data
        self.rt.lib = None

    def _upload(self, arr):
        a = self.mem.alloc(arr.size, arr.dtype)
        a[:] = arr.reshape(-1)
        return a.ctypes.data

    def view(self, b):
        t = b.root().tensor.arr
        o = b.root_offset()
        return t[o:o + b.numel].reshape(b.shape) if b.shape else t[o:o + 1].reshape(())

    def __call__(self, low, slots):
        self.calls += 1
        roots = [b for b in low.buffers if b.alias_of is None]
        for b in roots:  # bound only while probing, like ProbeRuntime
            if b.bid not in self.shims:
                self.shims[b.bid] = E._Shim(self.mem.alloc(b.numel, E.NPT[b.dtype]))
            b.tensor = self.shims[b.bid]
        try:
            if not self.loaded:
                for name, b in low.entry_inputs.items():
                    self.view(b)[...] = np.asarray(self.inputs[name]).reshape(b.shape)
                self.loaded = True
            for op in low.ops[self.done:]:
                op.prepare(self.rt)
                self.em.run_op(op)
                self.launches += 1
            self.done = len(low.ops)
            return {n: np.array(self.view(b)) for n, b in slots.items()}
        finally:
            for b in roots:
                b.tensor = None


def _incremental(prog, bundle, params, inputs):
    from paper_2509_02197_b200.api import _Known

    probe = _EmuProbe(inputs)
    lw = lower_gradient(prog, bundle, params, _check_inputs(prog, inputs, params), known=_Known(probe))
    em, view = E.execute(lw.low, inputs, lw.inputs, lw.seed_buf)
    return lw, view, probe


@pytest.mark.parametrize("cid", sorted(c for c in R2IDX["control_flow"] if c.startswith("loop_branch")))
def test_incremental_probe_lowers_once(cid):
    """ADVICE r1 (probe_lower O(T^2)): the decisions of a T-trip loop are
    resolved while lowering, each probe running only the launches emitted
    since the previous decision (T probes, each launch run once), with the
    reference's results."""
    prog, b = _r2_bundle("loop_branch")
    inputs, value, grads = _r2_case(cid)
    lw, view, probe = _incremental(prog, b, {}, inputs)
    assert rel_err(view(lw.outputs["value"]), value) <= 1e-12
    assert rel_err(view(lw.outputs["grad:t"]), grads["t"]) <= 1e-12
    assert probe.calls == len(lw.low.decisions) == 3
    # every probed launch ran once: no more launches than the unfinished list
    assert probe.launches <= len(lw.low.ops) + len(lw.low.decisions) * 4


@pytest.mark.parametrize("cid", sorted(c for c in R2IDX["control_flow"] if c.startswith("elem_branch")))
def test_branch_on_array_elements_snapshots_only_those_elements(cid):
    """Every trip of a 12-trip loop branches on x[i] (``idx``): each decision
    snapshots that one element (full-array snapshots pinned
    T x the array in HBM), re-evaluates from it alone, and the result is
    the reference's."""
    prog, b = _r2_bundle("elem_branch")
    inputs, value, grads = _r2_case(cid)
    lw, view, probe = _incremental(prog, b, {"N": 12}, inputs)
    assert rel_err(view(lw.outputs["value"]), value) <= 1e-12
    assert rel_err(view(lw.outputs["grad:x"]), grads["x"]) <= 1e-12
    decisions = lw.low.decisions
    assert probe.calls == len(decisions) == 12
    x = inputs["x"]
    for i, (slots, key_fn, key) in enumerate(decisions):
        assert {n: s.shape for n, s in slots.items()} == {"x": (1,)}
        assert float(view(lw.low.resolve(slots["x"]))[0]) == x[i]
        assert key is bool(x[i] < 1.0)
        assert key_fn({"x": np.array([0.5])}) is True and key_fn({"x": np.array([1.5])}) is False
    # the restart protocol gives the same launch list
    lw2, em, view2 = _emulate_probing(prog, b, {"N": 12}, inputs)
    assert len(lw2.low.ops) == len(lw.low.ops)
    assert rel_err(view2(lw2.outputs["grad:x"]), grads["x"]) <= 1e-12


# -- the reference CLI's plan artifacts (f1)


@pytest.mark.parametrize("cid", sorted(R2IDX["plans_cli"]))
def test_cli_plan_artifacts_give_the_same_plan(cid):
    """``gradflow plan --emit STEM --json`` + the ``gradflow diff`` manifest
    carry everything run_planned derives (checkpointing.py:917-942)."""
    meta = R2IDX["plans_cli"][cid]
    pb = plan_from_reference_artifacts(os.path.join(R2, "plans_cli", cid),
                                       os.path.join(R2, "plans_cli", cid + ".report.json"),
                                       os.path.join(os.path.dirname(GOLD), "..", meta["manifest"]))
    ref = load_plan(os.path.join(GOLD, "plans", cid))
    assert pb.keep == ref.keep
    assert pb.stored == ref.stored
    assert sorted(pb.forwarding) == sorted(ref.forwarding)
    assert dump_program(pb.forward) == dump_program(ref.forward)
    assert dump_program(pb.backward) == dump_program(ref.backward)


@pytest.mark.parametrize("cid", sorted(R2IDX["plans_cli"]))
def test_cli_plan_artifacts_replay_on_the_emulator(cid):
    meta = R2IDX["plans_cli"][cid]
    stem = os.path.join(R2, "plans_cli", cid)
    pb = load_plan(stem, manifest=os.path.join(os.path.dirname(GOLD), "..", meta["manifest"]))
    g = np.load(os.path.join(GOLD, "plans", cid + ".npz"))
    inputs = {k[3:]: g[k] for k in g.files if k.startswith("in:")}
    params = json.load(open(os.path.join(GOLD, "index.json")))["plans"][cid]["params"]
    shapes = _check_inputs(pb.forward, inputs, params)
    lw = lower_gradient(pb.forward, None, params, shapes, plan=pb)
    em, view = E.execute(lw.low, inputs, lw.inputs, lw.seed_buf)
    tol = tol_for(pb.forward)
    assert rel_err(view(lw.outputs["value"]), g["value"]) <= tol
    for k in (f[5:] for f in g.files if f.startswith("grad:")):
        got = view(lw.outputs["grad:" + k]) if "grad:" + k in lw.outputs else np.zeros_like(g["grad:" + k])
        assert rel_err(got, g["grad:" + k]) <= tol, k


# -- executable cache keys


def test_program_fingerprint_tracks_content_not_identity():
    prog, _ = _bundle("jacobi_2d")
    again = load_program(os.path.join(W.PROG_DIR, "jacobi_2d.fwd.json"))
    assert prog is not again and fingerprint(prog) == fingerprint(again)
    mutated = load_program(os.path.join(W.PROG_DIR, "jacobi_2d.fwd.json"))
    mutated.independents = ("A", "B")
    assert fingerprint(mutated) != fingerprint(prog)


# -- device memory timeline vs the reference simulate_memory (f4) -----------------

TIMELINES = json.load(open(os.path.join(R2, "timelines.json")))
_CFG_PLANS = json.load(open(os.path.join(W.PROG_DIR, "plans", "index.json")))
_GOLD_PLANS = json.load(open(os.path.join(GOLD, "index.json")))["plans"]


def _engine_timeline(cid):
    from paper_2509_02197_b200.runtime import memory_timeline, plan_arena

    if cid in _GOLD_PLANS:
        meta, pb = _GOLD_PLANS[cid], load_plan(os.path.join(GOLD, "plans", cid))
    else:
        meta, pb = _CFG_PLANS[cid], load_plan(os.path.join(W.PROG_DIR, "plans", cid))
    lw = lower_gradient(pb.forward, None, meta["params"], W.input_shapes(pb.forward, meta["params"]), plan=pb)
    low = lw.low
    roots = [b for b in low.buffers if b.alias_of is None]
    keep = {b.root().bid for b in lw.inputs.values()}
    if lw.seed_buf is not None:
        keep.add(lw.seed_buf.root().bid)
    outs = {b.root().bid for b in lw.outputs.values()}
    offsets, arena = plan_arena(low.ops, roots, keep, outs)
    return memory_timeline(low.ops, roots, keep, outs, offsets, low.buffers), arena


def _lifetimes(events):
    """array -> (first event index, last event index) from alloc/keep/
    recompute ... free events."""
    out = {}
    for k, ev in enumerate(events):
        kind, name = ev[0].split(" ", 1)
        if kind in ("alloc", "keep", "recompute", "snapshot"):
            out.setdefault(name, [k, None])
        elif kind == "free" and name in out:
            out[name][1] = k
    return {n: (a, len(events) if f is None else f) for n, (a, f) in out.items()}


@pytest.mark.parametrize("cid", sorted(TIMELINES))
def test_engine_memory_timeline_within_reference_simulation(cid):
    """The engine's arena residency, launch by launch (runtime.memory_timeline
    over the actual liveness placement), against the reference's
    simulate_memory for the same plan (verification.py:228-323): the peak and
    the arena never exceed the modelled peak t* (<= the budget), and any two
    arrays the engine holds at the same time are also both resident in the
    reference's timeline (the engine's lifetimes are nested in the model's;
    recompute scratch is inside the model's recompute spikes)."""
    tl, arena = _engine_timeline(cid)
    ref = TIMELINES[cid]
    ref_peak = max(p["peak_bytes"] for p in ref["paths"])
    assert tl["peak"] <= ref_peak and arena <= ref["model_peak_bytes"]
    assert tl["high_water"] <= arena
    if ref["limit_bytes"] is not None:
        assert arena <= ref["limit_bytes"]
    eng = _lifetimes([(e[0], e[1], e[2]) for e in tl["events"]])
    rl = _lifetimes(ref["paths"][0]["events"])
    # an engine buffer stands for every array sharing its storage (an elided
    # copy z1__grad = h1__grad lives in h1__grad's memory)
    names = {x: [n for n in tl["aliases"].get(x, [x]) if n in rl] or [x] for x in eng}
    both = sorted(x for x in eng if any(n in rl for n in names[x]))

    def ref_overlap(x, y):
        return any(rl[a][0] < rl[b][1] and rl[b][0] < rl[a][1] for a in names[x] if a in rl
                   for b in names[y] if b in rl)

    for i, x in enumerate(both):
        for y in both[i + 1:]:
            (ea, ef), (fa, ff) = eng[x], eng[y]
            if ea < ff and fa < ef:  # overlap in the engine
                assert ref_overlap(x, y), (x, y)


def test_batch_shape_follows_the_reference_rule():
    """The first input with extra leading dims fixes the batch shape
    (interpreter.py:161-169); shared inputs keep their declared shape;
    mismatched leading dims are a ShapeMismatch."""
    from paper_2509_02197_b200.api import batch_of
    from paper_2509_02197_b200.errors import ShapeMismatch

    prog, _ = _bundle("atax")
    params = {"M": 6, "N": 5}
    A, x = np.ones((6, 5)), np.ones((4, 3, 5, 1))
    assert batch_of(prog, {"A": A, "x": x}) == (4, 3)
    assert _check_inputs(prog, {"A": A, "x": x}, params, batch=(4, 3)) == {"A": (6, 5), "x": (5, 1)}
    with pytest.raises(ShapeMismatch):
        _check_inputs(prog, {"A": np.ones((2, 6, 5)), "x": x}, params, batch=(4, 3))
    assert batch_of(prog, {"A": A, "x": np.ones((5, 1))}) == ()


# -- sequential loop nests by hyperplanes (lowering.ProgramRun._wavefront) -------


def test_seidel_nest_lowers_to_two_wavefront_launches():
    """The corpus Gauss-Seidel nest (reference examples.py:159-182) runs as
    one hyperplane launch per direction instead of one launch per point;
    the emulated launch list reproduces the reference golden exactly and the
    reference op_count."""
    from conftest import load_case
    from paper_2509_02197_b200.lowering import WavefrontOp

    prog, b = _bundle("corpus_seidel_stencil")
    inputs, value, grads, op_count = load_case("corpus_seidel_stencil__N40_TSTEPS10")
    params = {"N": 40, "TSTEPS": 10}
    lw = lower_gradient(prog, b, params, _check_inputs(prog, inputs, params))
    waves = [op for op in lw.low.ops if isinstance(op, WavefrontOp)]
    assert len(waves) == 2 and len(lw.low.ops) <= 4
    assert waves[0].c == [2, 1, 1]  # forward: 2t + i + j
    em, view = E.execute(lw.low, inputs, lw.inputs, lw.seed_buf)
    assert rel_err(view(lw.outputs["value"]), value) <= 1e-13
    assert rel_err(view(lw.outputs["grad:A"]), grads["A"]) <= 1e-13
    assert lw.low.flops == op_count


def test_hyperplane_respects_every_dependence():
    from paper_2509_02197_b200.lowering import hyperplane

    # 2-D in-place recurrence x[i] = f(x[i-1]) inside a time loop: (t free, i)
    deps = [({1: 1}, frozenset({0})), ({1: -1}, frozenset({0})), ({1: 0}, frozenset({0}))]
    c = hyperplane([5, 7], deps)
    assert c is not None
    for d_t in range(-4, 5):
        for d_i in range(-6, 7):
            lexpos = d_t > 0 or (d_t == 0 and d_i > 0)
            if lexpos and d_i in (1, -1, 0):
                assert c[0] * d_t + c[1] * d_i >= 1
    # a dependence no small hyperplane can order: A[i] += B[j] over (i, j)
    # with i free inside j ... (every i conflicts with every other i)
    assert hyperplane([3, 50], [({}, frozenset({0, 1}))]) is None


def test_seidel_oracle_is_pinned_to_the_reference_golden():
    from conftest import load_case
    from oracle import stencil_ref as S

    inputs, value, _, _ = load_case("corpus_seidel_stencil__N40_TSTEPS10")
    assert rel_err(S.seidel_value({"N": 40, "TSTEPS": 10}, inputs["A"]), value) <= 1e-13
