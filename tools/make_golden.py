"""Generate the serialized programs and golden fixtures from the REFERENCE.

Runs only in the build container (imports /root/reference read-only):

    python tools/make_golden.py

Writes
  paper_2509_02197_b200/programs/<w>.fwd.json / .bwd.json / .fwdreq.json
      the reference forward program, its reverse program and forwarding
      manifest (the exact files ``gradflow diff`` emits, cli.py:211-243);
  tests/golden/<case>.npz
      inputs (default_rng(seed).uniform(0.4, 1.6), descriptor order, the
      reference ``sample_inputs`` rule, verification.py:157-175), the
      reference gradient()'s value / grads / op_count;
  tests/golden/plans/<case>.{fwd,bwd,plan}.json + .npz
      reference plan() results at several budgets and run_planned() outputs;
  tests/golden/infeasible.json
      Infeasible.min_peak_bytes of the literal C2 budget (25 % of store-all).
"""
from __future__ import annotations

import json
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)
sys.path.insert(0, REPO)
warnings.simplefilter("ignore")

import gradflow.examples as ref_examples  # noqa: E402
from gradflow import errors as ref_errors  # noqa: E402
from gradflow.autodiff import build_backward, gradient  # noqa: E402
from gradflow.checkpointing import plan, run_planned  # noqa: E402
from gradflow.frontend import serialize_program  # noqa: E402
from gradflow.verification import sample_inputs  # noqa: E402

from workloads_ref import WORKLOADS  # noqa: E402

from paper_2509_02197_b200.api import as_plan, save_plan  # noqa: E402
from paper_2509_02197_b200.ir import adopt  # noqa: E402
from paper_2509_02197_b200.workloads import SMALL_PARAMS, make_inputs  # noqa: E402

PROG_DIR = os.path.join(REPO, "paper_2509_02197_b200", "programs")
GOLD = os.path.join(REPO, "tests", "golden")
PLANS = os.path.join(GOLD, "plans")
MIB = 1 << 20


def save_programs(name, program):
    bundle = build_backward(program)
    stem = os.path.join(PROG_DIR, name)
    with open(stem + ".fwd.json", "w") as f:
        f.write(serialize_program(program))
    with open(stem + ".bwd.json", "w") as f:
        f.write(serialize_program(bundle.backward))
    manifest = {
        "required": sorted([d, v] for d, v in bundle.required),
        "entries": [
            {"name": e.name, "data": e.data,
             "candidates": [{"version": c.version, "directives": [list(d) for d in c.directives]}
                            for c in e.candidates]}
            for e in sorted(bundle.forwarding.values(), key=lambda e: e.name)
        ],
    }
    with open(stem + ".fwdreq.json", "w") as f:
        json.dump(manifest, f, indent=2)
        f.write("\n")
    return bundle


def case_id(name, params):
    return name + "__" + "_".join(f"{k}{v}" for k, v in params.items())


def inputs_for(name, program, params, seed):
    if name.startswith("corpus_"):
        return sample_inputs(program, params, np.random.default_rng(seed))
    return make_inputs(name, adopt(program), params, seed)


def save_case(name, program, bundle, params, seed=0):
    inputs = inputs_for(name, program, params, seed)
    t0 = time.perf_counter()
    res = gradient(program, inputs, params, bundle=bundle)
    dt = time.perf_counter() - t0
    arrays = {f"in:{k}": v for k, v in inputs.items()}
    arrays["value"] = np.asarray(res.value)
    for k, v in res.grads.items():
        arrays[f"grad:{k}"] = np.asarray(v)
    arrays["op_count"] = np.asarray(res.forward.op_count + res.backward.op_count, dtype=np.int64)
    cid = case_id(name, params)
    np.savez_compressed(os.path.join(GOLD, cid + ".npz"), **arrays)
    meta = {"workload": name, "params": params, "seed": seed, "ref_seconds": dt}
    print(f"  {cid}: value={float(np.asarray(res.value)):.12g} ({dt:.2f}s)")
    return cid, meta


def save_plan_case(name, program, params, limit_mib, tag, seed=0):
    result = plan(program, limit_mib, params)
    pb = as_plan(result)
    cid = f"{case_id(name, params)}__{tag}"
    save_plan(pb, os.path.join(PLANS, cid))
    inputs = inputs_for(name if name in SMALL_PARAMS else "corpus_" + name, program, params, seed)
    res = run_planned(result, inputs, params)
    arrays = {f"in:{k}": v for k, v in inputs.items()}
    arrays["value"] = np.asarray(res.value)
    for k, v in res.grads.items():
        arrays[f"grad:{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(PLANS, cid + ".npz"), **arrays)
    decisions = [v["decision"] for v in result.report["values"]]
    print(f"  plan {cid}: limit={limit_mib} decisions={decisions} peak={result.solution.t_star}")
    return cid, {"workload": name, "params": params, "limit_mib": limit_mib,
                 "assignment": list(result.solution.assignment), "t_star": result.solution.t_star,
                 "objective_flops": result.solution.objective_flops, "decisions": decisions}


def budgets(program, params):
    """store-all peak, floor, and floor + 25 % of the gap."""
    full = plan(program, None, params)
    store_all = full.solution.t_star
    try:
        plan(program, 0.0, params)
        floor = 0
    except ref_errors.Infeasible as exc:
        floor = exc.min_peak_bytes
    return store_all, floor


def main():
    os.makedirs(PROG_DIR, exist_ok=True)
    os.makedirs(PLANS, exist_ok=True)
    index = {"cases": {}, "plans": {}, "examples": {}}
    for name, build in WORKLOADS.items():
        print(name)
        program = build()
        bundle = save_programs(name, program)
        for params in SMALL_PARAMS[name]:
            cid, meta = save_case(name, program, bundle, params)
            index["cases"][cid] = meta
    # plans with real ILP variables: softmax, mlp, Listing-1 chain
    plan_targets = [("softmax", WORKLOADS["softmax"](), {"R": 64, "SM": 32}),
                    ("mlp", WORKLOADS["mlp"](), {"NB": 8, "C": 16, "S0": 24, "S1": 12, "S2": 10}),
                    ("scaled_product_chain", ref_examples.build("scaled_product_chain"), {"N": 16})]
    for name, program, params in plan_targets:
        store_all, floor = budgets(program, params)
        for tag, limit in (("none", None), ("storeall", store_all / MIB),
                           ("tight", (floor + 0.25 * (store_all - floor)) / MIB), ("floor", floor / MIB)):
            try:
                cid, meta = save_plan_case(name, program, params, limit, tag)
                meta.update(store_all=store_all, floor=floor)
                index["plans"][cid] = meta
            except ref_errors.Infeasible as exc:
                print(f"  plan {name} {tag}: infeasible ({exc.min_peak_bytes})")
    # literal config 2: 25 % of store-all for the linear stencils
    inf = {}
    for name, params in (("jacobi_2d", {"N": 700, "TSTEPS": 200}), ("heat_3d", {"N": 70, "TSTEPS": 100})):
        program = WORKLOADS[name]()
        full = plan(program, None, params)
        limit = 0.25 * full.solution.t_star / MIB
        try:
            plan(program, limit, params)
            inf[name] = {"params": params, "limit_mib": limit, "feasible": True}
        except ref_errors.Infeasible as exc:
            inf[name] = {"params": params, "limit_mib": limit, "store_all": full.solution.t_star,
                         "min_peak_bytes": exc.min_peak_bytes, "message": str(exc)}
        print("  C2", name, inf[name])
    with open(os.path.join(GOLD, "infeasible.json"), "w") as f:
        json.dump(inf, f, indent=2)
    # the reference's own corpus (examples.py:306-338) at its default params
    for name in ref_examples.EXAMPLES:
        program = ref_examples.build(name)
        params = ref_examples.DEFAULT_PARAMS[name]
        bundle = save_programs("corpus_" + name, program)
        cid, meta = save_case("corpus_" + name, program, bundle, params, seed=101)
        index["examples"][cid] = meta
    with open(os.path.join(GOLD, "index.json"), "w") as f:
        json.dump(index, f, indent=2)


if __name__ == "__main__":
    main()
