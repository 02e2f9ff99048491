"""Host lowering checked on the CPU: the launch list the engine would run,
executed by the descriptor emulator (tests/emulator.py), must reproduce the
reference goldens; plus the structural properties the B200 design relies on
(clear folding, tape aliasing, op_count, static errors)."""
import os

import numpy as np
import pytest

import emulator as E
from conftest import GOLD, golden_index, load_case, rel_err, tol_for
from paper_2509_02197_b200 import workloads as W
from paper_2509_02197_b200.api import _check_inputs, load_bundle, load_plan, lower_gradient
from paper_2509_02197_b200.errors import DomainError, OutOfBounds, UnsupportedConstruct
from paper_2509_02197_b200.ir import load_program
from paper_2509_02197_b200.lowering import FillOp, NeedValues, StencilOp
from oracle import interp as O

IDX = golden_index()


def _bundle(name):
    stem = os.path.join(W.PROG_DIR, name)
    return load_program(stem + ".fwd.json"), load_bundle(stem + ".bwd.json", stem + ".fwdreq.json")


def _emulate(prog, bundle, params, inputs, plan=None):
    shapes = _check_inputs(prog, inputs, params)
    lw = lower_gradient(prog, bundle, params, shapes, plan=plan)
    em, view = E.execute(lw.low, inputs, lw.inputs, lw.seed_buf)
    return lw, em, view


def _check(lw, view, prog, value, grads):
    tol = tol_for(prog)
    assert rel_err(view(lw.outputs["value"]), value) <= tol
    for k, ref in grads.items():
        got = view(lw.outputs["grad:" + k]) if "grad:" + k in lw.outputs else np.zeros_like(ref)
        assert rel_err(got, ref) <= tol, k


CASES = sorted(IDX["cases"]) + sorted(c for c in IDX["examples"] if "branchy" not in c)


@pytest.mark.parametrize("cid", CASES)
def test_lowered_launch_list_matches_reference(cid):
    meta = IDX["cases"].get(cid) or IDX["examples"][cid]
    prog, b = _bundle(meta["workload"])
    inputs, value, grads, op_count = load_case(cid)
    lw, em, view = _emulate(prog, b, meta["params"], inputs)
    _check(lw, view, prog, value, grads)
    assert lw.low.flops == op_count  # reference dynamic op_count (interpreter.py:426)
    assert int(em.err[0]) == 0


@pytest.mark.parametrize("cid", sorted(IDX["plans"]))
def test_lowered_planned_replay(cid):
    meta = IDX["plans"][cid]
    pb = load_plan(os.path.join(GOLD, "plans", cid))
    inputs, value, grads, _ = load_case(cid, "plans")
    lw, em, view = _emulate(pb.forward, None, meta["params"], inputs, plan=pb)
    _check(lw, view, pb.forward, value, grads)


def test_stencil_timestep_is_one_fused_launch_with_clears_folded():
    """heat_3d: each timestep (2 forward sweeps, or 2 adjoint gather sweeps
    with their `_z` clears folded) is ONE fused star-pair launch; no
    separate clear passes; dead intermediates are not written back."""
    from paper_2509_02197_b200.lowering import StarPairOp

    prog, b = _bundle("heat_3d")
    params = {"N": 10, "TSTEPS": 5}
    inputs = W.make_inputs("heat_3d", prog, params, 0)
    lw = lower_gradient(prog, b, params, _check_inputs(prog, inputs, params), fuse_small=True)
    pairs = [op for op in lw.low.ops if isinstance(op, StarPairOp)]
    assert len(pairs) == 2 * (params["TSTEPS"] - 1)
    assert not any(isinstance(op, (FillOp, StencilOp)) for op in lw.low.ops)
    fwd, bwd = pairs[: len(pairs) // 2], pairs[len(pairs) // 2:]
    # between timesteps only the boundary shell of the intermediate (B, B__grad) is live
    assert all(p.xwrite and p.dead is not None for p in fwd[:-1] + bwd[:-1])
    assert not fwd[-1].xwrite and not bwd[-1].xwrite  # never read again, not observed
    assert all(p.b.clear_mode in (1, 2) for p in bwd)


def test_unfused_launch_list_matches_too(monkeypatch):
    monkeypatch.setenv("GFB_FUSE", "0")
    prog, b = _bundle("heat_3d")
    cid = "heat_3d__N8_TSTEPS3"
    inputs, value, grads, _ = load_case(cid)
    lw, em, view = _emulate(prog, b, IDX["cases"][cid]["params"], inputs)
    assert any(isinstance(op, StencilOp) for op in lw.low.ops)
    _check(lw, view, prog, value, grads)


def test_tape_snapshot_is_aliased_when_never_overwritten():
    prog, b = _bundle("atax")
    params = {"M": 6, "N": 5}
    inputs = W.make_inputs("atax", prog, params, 0)
    lw = lower_gradient(prog, b, params, _check_inputs(prog, inputs, params), fuse_small=True)
    slots = list(lw.tape.values.values())
    assert slots and all(s.alias_of is not None for s in slots)


def test_out_of_bounds_is_static():
    prog, b = _bundle("jacobi_2d")
    params = {"N": 6, "TSTEPS": 3}
    inputs = W.make_inputs("jacobi_2d", prog, {"N": 6, "TSTEPS": 3}, 0)
    # declared shape N=6 but a map reaching N: simulate with a wrong binding
    with pytest.raises(OutOfBounds):
        lower_gradient(prog, b, {"N": 6, "TSTEPS": 3}, {"A": (5, 5), "B": (5, 5)})


def test_domain_error_bit_from_emulated_kernel():
    prog, b = _bundle("softmax")
    params = {"R": 3, "SM": 4}
    inputs = W.make_inputs("softmax", prog, params, 0)
    inputs["x"][:] = -200.0  # exp underflows to 0 -> row sum 0 -> div by zero
    lw, em, view = _emulate(prog, b, params, inputs)
    assert int(em.err[0]) & 0x1


def _emulate_probing(prog, bundle, params, inputs):
    """lower_gradient with the api's probe loop, every probe run (and the
    final launch list) on the emulator instead of the device."""
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
    return lw, em, view, known


def test_data_dependent_branch_needs_a_probe():
    prog, b = _bundle("corpus_branchy_scale")
    params = {"n": 8}
    inputs = {"X": np.ones(8), "s": np.array(0.3)}
    with pytest.raises(NeedValues) as ei:
        lower_gradient(prog, b, params, _check_inputs(prog, inputs, params))
    assert sorted(ei.value.slots) == ["s"]


def test_data_dependent_branch_matches_reference_golden():
    """Reference interpreter.py:342-347: the condition reads the scalar input
    s; the golden draws s = 1.57, so the 'high' (sin) arm runs."""
    prog, b = _bundle("corpus_branchy_scale")
    inputs, value, grads, op_count = load_case("corpus_branchy_scale__n8")
    lw, em, view, known = _emulate_probing(prog, b, {"n": 8}, inputs)
    _check(lw, view, prog, value, grads)
    assert lw.low.flops == op_count
    assert len(known) == 1 and len(lw.low.decisions) == 1
    slots, key_fn, key = lw.low.decisions[0]
    assert key is False
    # the recorded decision re-evaluates from the final run's snapshot
    assert key_fn({n: np.array(view(lw.low.resolve(s))) for n, s in slots.items()}) is False
    assert key_fn({"s": np.array(0.3)}) is True


@pytest.mark.parametrize("s", [0.3, 0.5, 0.9])
def test_data_dependent_branch_both_arms_match_oracle(s):
    prog, b = _bundle("corpus_branchy_scale")
    params = {"n": 8}
    rng = np.random.default_rng(3)
    inputs = {"X": rng.uniform(0.4, 1.6, 8), "s": np.array(s)}
    lw, em, view, _ = _emulate_probing(prog, b, params, inputs)
    v, g, _ = O.gradient(prog, b.backward, b.forwarding, b.required, inputs, params)
    _check(lw, view, prog, v, g)
    want = 2.0 if s < 0.5 else np.cos(inputs["X"])
    assert np.allclose(view(lw.outputs["grad:X"]), want, rtol=1e-14, atol=0)


def _scalar_loop():
    import json

    rec = json.load(open(os.path.join(GOLD, "scalar_trip_loop.json")))
    return load_program(os.path.join(GOLD, "scalar_trip_loop.fwd.json")), rec


def _emulate_forward_probing(prog, params, inputs):
    from paper_2509_02197_b200.api import _init_env
    from paper_2509_02197_b200.ir import number_writes
    from paper_2509_02197_b200.lowering import Lowering, ProgramRun

    shapes = _check_inputs(prog, inputs, params)
    known = []
    while True:
        low = Lowering(known=known)
        env, ins = _init_env(low, prog, shapes, "")
        low.entry_inputs = ins
        try:
            ProgramRun(low, prog, params, env, versions=number_writes(prog)).run()
            break
        except NeedValues as nv:
            low.finish(list(nv.slots.values()))
            _, pview = E.execute(low, inputs, ins)
            known.append({n: np.array(pview(low.resolve(b))) for n, b in nv.slots.items()})
    low.finish(list(env.values()))
    _, view = E.execute(low, inputs, ins)
    return low, env, view, known


def test_scalar_trip_count_loop_matches_reference_forward():
    """Loop header bound to a scalar input (reference interpreter.py:210-219):
    the trip count comes from a probe of k, then the loop unrolls."""
    prog, rec = _scalar_loop()
    x = np.array(rec["X"])
    for run in rec["runs"]:
        low, env, view, known = _emulate_forward_probing(prog, rec["params"], {"X": x, "k": np.array(run["k"])})
        assert len(known) == 1
        assert abs(float(view(low.resolve(env["O"]))) - run["value"]) <= 1e-10
        assert np.allclose(view(low.resolve(env["Y"])), run["Y"], rtol=1e-12, atol=0)
        assert low.flops == run["op_count"]
    assert rec["non_integer"] == "DomainError"
    with pytest.raises(DomainError):
        _emulate_forward_probing(prog, rec["params"], {"X": x, "k": np.array(2.5)})


@pytest.mark.parametrize("name", ["atax", "bicg"])
def test_matvec_pairs_and_rank2_fuse_and_match_goldens(name):
    """Both matrix-vector pairs (forward and adjoint) become one-pass
    MatvecPairOps and the two outer-product adjoints one Rank2Op; the fused
    list (emulated as its parts, in order) still reproduces the reference."""
    from paper_2509_02197_b200.lowering import MatmulOp, MatvecPairOp, Rank2Op

    prog, b = _bundle(name)
    cid = f"{name}__M40_N33"
    inputs, value, grads, _ = load_case(cid)
    lw, em, view = _emulate(prog, b, IDX["cases"][cid]["params"], inputs)
    ops = lw.low.ops
    assert sum(isinstance(op, MatvecPairOp) for op in ops) == 2
    assert sum(isinstance(op, Rank2Op) for op in ops) == 1
    assert not any(isinstance(op, MatmulOp) for op in ops)
    if name == "atax":
        assert [op.chain for op in ops if isinstance(op, MatvecPairOp)] == [True, True]
    _check(lw, view, prog, value, grads)


def test_matvec_pairing_respects_an_intervening_write():
    """A write to the matrix between the two nodes blocks the pairing."""
    from paper_2509_02197_b200.lowering import FillOp, Lowering, MatmulOp, MatvecPairOp

    low = Lowering()
    A = low.new_buffer("A", (8, 8), "real64", fresh=False)
    x = low.new_buffer("x", (8, 1), "real64", fresh=False)
    t = low.new_buffer("t", (8, 1), "real64", fresh=False)
    y = low.new_buffer("y", (8, 1), "real64", fresh=False)
    low.ops = [MatmulOp(A, x, t, False, False, 8, 1, 8, False), FillOp(A, ((0, 8), (0, 8)), 1.0),
               MatmulOp(A, t, y, True, False, 8, 1, 8, False)]
    low._fuse_matvec_pairs()
    assert not any(isinstance(op, MatvecPairOp) for op in low.ops)
    low.ops = [MatmulOp(A, x, t, False, False, 8, 1, 8, False), MatmulOp(A, t, y, True, False, 8, 1, 8, False)]
    low._fuse_matvec_pairs()
    assert [type(op).__name__ for op in low.ops] == ["MatvecPairOp"] and low.ops[0].chain
