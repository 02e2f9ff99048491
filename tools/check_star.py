"""Quick GPU check of the star-pair kernels (TMA and L1 variants) against the
oracle on small heat_3d / jacobi_2d cases."""
import os
import sys

os.environ.setdefault("GFB_SMALL_FUSE_BYTES", "0")  # exercise the fused kernels at small sizes

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import interp as O  # noqa: E402
from paper_2509_02197_b200 import gradient, workloads as W  # noqa: E402
from paper_2509_02197_b200.api import clear_cache  # noqa: E402

cases = [("heat_3d", {"N": 40, "TSTEPS": 5}), ("heat_3d", {"N": 66, "TSTEPS": 4}), ("jacobi_2d", {"N": 100, "TSTEPS": 6}),
         ("heat_3d", {"N": 35, "TSTEPS": 3})]
bad = 0
for name, params in cases:
    prog, b = W.load(name)
    inp = W.make_inputs(name, prog, params, 0)
    v, g, _ = O.gradient(prog, b.backward, b.forwarding, b.required, inp, params)
    for tma in ("1", "0"):
        if tma == "0":
            os.environ["GFB_NO_TMA"] = "1"
        else:
            os.environ.pop("GFB_NO_TMA", None)
        clear_cache()
        res = gradient(prog, inp, params, bundle=b)
        ev = abs(float(res.value) - float(v)) / abs(float(v))
        eg = float(np.max(np.abs(res.grads["A"] - g["A"]) / np.maximum(1, np.abs(g["A"]))))
        ok = ev < 1e-10 and eg < 1e-10
        bad += not ok
        print(f"{name} {params} tma={tma}: value err {ev:.2e} grad err {eg:.2e} {'OK' if ok else 'FAIL'}")
sys.exit(1 if bad else 0)
