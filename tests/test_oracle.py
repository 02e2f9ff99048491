"""Pin the oracle (oracle/interp.py) against golden vectors produced by the
real reference (tests/golden, tools/make_golden.py) and against the survey's
full-size C1 golden."""
import json
import os

import numpy as np
import pytest

from conftest import GOLD, golden_index, load_case, rel_err, tol_for
from oracle import interp as O
from paper_2509_02197_b200 import workloads as W
from paper_2509_02197_b200.api import load_bundle, load_plan
from paper_2509_02197_b200.ir import load_program

IDX = golden_index()
PROG = W.PROG_DIR


def _bundle(name):
    stem = os.path.join(PROG, name)
    return load_program(stem + ".fwd.json"), load_bundle(stem + ".bwd.json", stem + ".fwdreq.json")


@pytest.mark.parametrize("cid", sorted(IDX["cases"]) + sorted(c for c in IDX["examples"] if "seidel" not in c))
def test_oracle_matches_reference_goldens(cid):
    meta = IDX["cases"].get(cid) or IDX["examples"][cid]
    prog, b = _bundle(meta["workload"])
    inputs, value, grads, op_count = load_case(cid)
    v, g, ops = O.gradient(prog, b.backward, b.forwarding, b.required, inputs, meta["params"])
    tol = tol_for(prog)
    assert rel_err(v, value) <= tol
    for k in grads:
        assert rel_err(g[k], grads[k]) <= tol, k
    assert ops == op_count


@pytest.mark.parametrize("cid", sorted(IDX["plans"]))
def test_oracle_planned_replay(cid):
    meta = IDX["plans"][cid]
    pb = load_plan(os.path.join(GOLD, "plans", cid))
    inputs, value, grads, _ = load_case(cid, "plans")
    v, g, _ = O.run_planned(pb, inputs, meta["params"])
    tol = tol_for(pb.forward)
    assert rel_err(v, value) <= tol
    for k in grads:
        assert rel_err(g[k], grads[k]) <= tol, k


def test_oracle_full_size_c1_survey_golden():
    """reference gradient at C1 (N=200, TSTEPS=50, A then B from
    default_rng(0).uniform(0.4,1.6)): value 40061.09429461688,
    sum(A__grad) 38211.744030772315, A__grad[100,100] = 1.0."""
    prog, b = _bundle("jacobi_2d")
    params = {"N": 200, "TSTEPS": 50}
    inputs = W.make_inputs("jacobi_2d", prog, params, 0)
    v, g, _ = O.gradient(prog, b.backward, b.forwarding, b.required, inputs, params)
    assert abs(float(v) - 40061.09429461688) / 40061.09429461688 < 1e-12
    assert abs(float(g["A"].sum()) - 38211.744030772315) / 38211.744030772315 < 1e-12
    assert abs(float(g["A"][100, 100]) - 1.0) < 1e-12
