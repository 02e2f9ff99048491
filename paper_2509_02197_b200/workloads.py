"""Built-in workloads: the BASELINE.json configs as reference-emitted programs.

The programs under ``programs/`` are the reference's own artifacts for the
Appendix-A encodings: ``<w>.fwd.json`` (forward program),
``<w>.bwd.json`` + ``<w>.fwdreq.json`` (the ``gradflow diff`` output of the
reference AD, cli.py:211-243). They are regenerated from the reference by
``tools/make_golden.py``; the engine only reads them.

Inputs follow the reference ``sample_inputs`` rule (verification.py:157-175):
``default_rng(seed).uniform(0.4, 1.6)`` per input descriptor in declaration
order, in the declared precision. One deviation, stated in DESIGN.md: the mlp
weight matrices are divided by their fan-in after sampling, because with
all-positive O(1) weights the 3-layer logits overflow exp() in fp32 and the
reference itself returns NaN.
"""
from __future__ import annotations

import os

import numpy as np

from .ir import eval_int, load_program

PROG_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "programs")

NAMES = ("jacobi_2d", "heat_3d", "gemm", "atax", "bicg", "softmax", "mlp", "conv2d_bias")

# BASELINE.json configs at the sizes they are quoted on (DESIGN.md pins the
# ones NPBench does not fix).
CONFIGS = {
    "C1/jacobi_2d": ("jacobi_2d", {"N": 200, "TSTEPS": 50}),
    "C2/jacobi_2d": ("jacobi_2d", {"N": 700, "TSTEPS": 200}),
    "C2/heat_3d": ("heat_3d", {"N": 70, "TSTEPS": 100}),
    "C3/gemm": ("gemm", {"NI": 4000, "NJ": 4000, "NK": 4000}),
    "C3/atax": ("atax", {"M": 4000, "N": 4000}),
    "C3/bicg": ("bicg", {"M": 4000, "N": 4000}),
    "C4/softmax": ("softmax", {"R": 64 * 16 * 128, "SM": 128}),
    "C4/mlp": ("mlp", {"NB": 64, "C": 512, "S0": 4096, "S1": 4096, "S2": 1024}),
    "C4/conv2d_bias": ("conv2d_bias", {"NB": 64, "H": 64, "W": 64, "CI": 16, "CO": 32, "K": 3}),
    "C5/heat_3d": ("heat_3d", {"N": 512, "TSTEPS": 100}),
}

# sizes at which the reference interpreter finishes in seconds (goldens)
SMALL_PARAMS = {
    "jacobi_2d": [{"N": 12, "TSTEPS": 4}, {"N": 40, "TSTEPS": 6}, {"N": 7, "TSTEPS": 1}, {"N": 9, "TSTEPS": 2}],
    "heat_3d": [{"N": 8, "TSTEPS": 3}, {"N": 6, "TSTEPS": 2}],
    "gemm": [{"NI": 7, "NJ": 5, "NK": 6}, {"NI": 32, "NJ": 24, "NK": 40}],
    "atax": [{"M": 6, "N": 5}, {"M": 40, "N": 33}],
    "bicg": [{"M": 6, "N": 5}, {"M": 40, "N": 33}],
    "softmax": [{"R": 6, "SM": 5}, {"R": 64, "SM": 32}],
    "mlp": [{"NB": 4, "C": 3, "S0": 6, "S1": 5, "S2": 4}, {"NB": 8, "C": 16, "S0": 24, "S1": 12, "S2": 10}],
    "conv2d_bias": [{"NB": 2, "H": 6, "W": 5, "CI": 2, "CO": 3, "K": 3}],
}

_FAN_IN = {"W1": "C", "W2": "S0", "W3": "S1"}


def load(name: str):
    """(forward Program, Bundle) of a built-in workload."""
    from .api import load_bundle

    stem = os.path.join(PROG_DIR, name)
    return load_program(stem + ".fwd.json"), load_bundle(stem + ".bwd.json", stem + ".fwdreq.json")


def input_shapes(program, params) -> dict:
    return {n: tuple(eval_int(s, params) for s in d.shape)
            for n, d in program.descriptors.items() if d.role == "input"}


def make_inputs(name: str, program, params: dict, seed: int = 0) -> dict:
    rng = np.random.default_rng(seed)
    out = {}
    for d in program.descriptors.values():
        if d.role != "input":
            continue
        shape = tuple(eval_int(s, params) for s in d.shape)
        dt = np.float32 if d.element_kind == "real32" else np.float64
        out[d.name] = rng.uniform(0.4, 1.6, shape).astype(dt)
    if name == "mlp":
        for w, fan in _FAN_IN.items():
            out[w] = (out[w] / np.float32(params[fan])).astype(np.float32)
    return out
