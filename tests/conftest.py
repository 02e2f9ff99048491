import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GOLD = os.path.join(HERE, "golden")
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

REF_SRC = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(REF_SRC)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libgfb.so")
    config.addinivalue_line("markers", "ref: needs the read-only reference checkout (build container only)")


def pytest_collection_modifyitems(config, items):
    if not HAVE_REF:
        skip = pytest.mark.skip(reason="reference checkout not present on this machine")
        for it in items:
            if "ref" in it.keywords:
                it.add_marker(skip)


def golden_index():
    with open(os.path.join(GOLD, "index.json")) as f:
        return json.load(f)


def load_case(cid, sub=""):
    g = np.load(os.path.join(GOLD, sub, cid + ".npz"))
    inputs = {k[3:]: g[k] for k in g.files if k.startswith("in:")}
    grads = {k[5:]: g[k] for k in g.files if k.startswith("grad:")}
    op_count = int(g["op_count"]) if "op_count" in g.files else None
    return inputs, g["value"], grads, op_count


def rel_err(got, ref):
    """reference compare_gradients metric |a-b| / max(1, |b|) (verification.py:131-141)."""
    a = np.asarray(got, dtype=np.float64).reshape(-1)
    b = np.asarray(ref, dtype=np.float64).reshape(-1)
    if a.shape != b.shape:
        return float("inf")
    if not a.size:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


def tol_for(program):
    """north_star tolerance: rtol 1e-10 (fp64), 1e-5 (fp32)."""
    kinds = {d.element_kind for d in program.descriptors.values()}
    return 1e-5 if "real32" in kinds else 1e-10
