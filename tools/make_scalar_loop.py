"""Golden fixture for a loop whose trip count is a scalar input (reference
interpreter.py:210-219, _header_bindings): the forward program and the
reference run_forward values at two trip counts. The reference's own AD
rejects such headers in the backward program (build_backward: "loop init
uses ['k']"), so only the forward path is pinned. Run in the build
container (reads /root/reference)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from gradflow.frontend import ProgramBuilder, serialize_program  # noqa: E402
from gradflow.interpreter import run_forward  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")

b = ProgramBuilder(("n",))
b.array("X", ("n",), role="input", kind="real64")
b.scalar("k", role="input", kind="real64")
b.array("Y", ("n",), kind="real64")
b.scalar("O", role="output", kind="real64")
with b.state("init") as st:
    st.library("ew_unary", {"x": "X"}, {"y": "Y"}, op="copy")
with b.loop("t", "0", "k", label="L"):
    with b.state("body") as st:
        st.library("ew_unary", {"x": "Y"}, {"y": "Y"}, op="sin")
with b.state("tail") as s:
    s.library("reduce_sum", {"x": "Y"}, {"y": "O"})
prog = b.finish("O", ["X"])
with open(os.path.join(OUT, "scalar_trip_loop.fwd.json"), "w") as f:
    f.write(serialize_program(prog))
x = np.random.default_rng(0).uniform(0.4, 1.6, 6)
rec = {"params": {"n": 6}, "X": x.tolist(), "runs": []}
for k in (0.0, 2.0, 5.0):
    r = run_forward(prog, {"X": x, "k": np.array(k)}, {"n": 6})
    rec["runs"].append({"k": k, "value": float(r.value), "Y": np.asarray(r.env["Y"]).tolist(),
                        "op_count": int(r.op_count)})
try:
    run_forward(prog, {"X": x, "k": np.array(2.5)}, {"n": 6})
except Exception as e:  # noqa: BLE001
    rec["non_integer"] = type(e).__name__
with open(os.path.join(OUT, "scalar_trip_loop.json"), "w") as f:
    json.dump(rec, f, indent=1)
print(rec["non_integer"], [r["value"] for r in rec["runs"]])
