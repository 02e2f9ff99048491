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
