"""Config encodings built with the REFERENCE's own
ProgramBuilder (``gradflow.frontend.ProgramBuilder``, reference
``pkg/src/gradflow/frontend.py:417-555``).

This module runs only in the build container, where ``/root/reference`` is
importable; it is the generator for the serialized programs under
``paper_2509_02197_b200/programs/`` and the golden fixtures under
``tests/golden/``. Nothing on the GPU box imports it.

Each builder returns a validated reference ``Program``. ``CONFIG_PARAMS``
pins the sizes the configs are quoted on (BASELINE.json ``configs``); where
NPBench sizes are not vendored the values are pinned here explicitly and
documented in DESIGN.md.
"""
from __future__ import annotations

import sys

sys.path.insert(0, "/root/reference/pkg/src")

from gradflow.frontend import ProgramBuilder  # noqa: E402


def _stencil_body_2d(src):
    return {
        "cc": (src, ("i", "j")),
        "ww": (src, ("i", "(sub j 1)")),
        "ee": (src, ("i", "(add j 1)")),
        "ss": (src, ("(add i 1)", "j")),
        "nn": (src, ("(sub i 1)", "j")),
    }


def jacobi_2d():
    """NPBench jacobi_2d: two 5-point sweeps per timestep, t in [1, TSTEPS)."""
    b = ProgramBuilder(("N", "TSTEPS"))
    b.array("A", ("N", "N"), role="input", kind="real64")
    b.array("B", ("N", "N"), role="input", kind="real64")
    b.scalar("O", role="output", kind="real64")
    rng = (("1", "(sub N 1)", "1"), ("1", "(sub N 1)", "1"))
    body = "(mul 0.2 (add (add (add (add cc ww) ee) ss) nn))"
    with b.loop("t", "1", "TSTEPS", label="time"):
        with b.state("step") as s:
            def sweep_b(inner):
                inner.tasklet(ins=_stencil_body_2d("A"), outs={"o": ("B", ("i", "j"))}, body={"o": body})

            def sweep_a(inner):
                inner.tasklet(ins=_stencil_body_2d("B"), outs={"o": ("A", ("i", "j"))}, body={"o": body})

            s.map_node(("i", "j"), rng, sweep_b)
            s.map_node(("i", "j"), rng, sweep_a)
    with b.state("collect") as s:
        s.library("reduce_sum", {"x": "A"}, {"y": "O"})
    return b.finish("O", ["A"])


def _stencil_body_3d(src):
    return {
        "cc": (src, ("i", "j", "k")),
        "ip": (src, ("(add i 1)", "j", "k")),
        "im": (src, ("(sub i 1)", "j", "k")),
        "jp": (src, ("i", "(add j 1)", "k")),
        "jm": (src, ("i", "(sub j 1)", "k")),
        "kp": (src, ("i", "j", "(add k 1)")),
        "km": (src, ("i", "j", "(sub k 1)")),
    }


HEAT_BODY = (
    "(add (add (add cc (mul 0.125 (add (sub ip (mul 2.0 cc)) im)))"
    " (mul 0.125 (add (sub jp (mul 2.0 cc)) jm)))"
    " (mul 0.125 (add (sub kp (mul 2.0 cc)) km)))"
)


def heat_3d():
    """NPBench heat_3d: two 7-point sweeps per timestep, t in [1, TSTEPS)."""
    b = ProgramBuilder(("N", "TSTEPS"))
    b.array("A", ("N", "N", "N"), role="input", kind="real64")
    b.array("B", ("N", "N", "N"), role="input", kind="real64")
    b.scalar("O", role="output", kind="real64")
    rng = (("1", "(sub N 1)", "1"),) * 3
    with b.loop("t", "1", "TSTEPS", label="time"):
        with b.state("step") as s:
            def sweep_b(inner):
                inner.tasklet(ins=_stencil_body_3d("A"), outs={"o": ("B", ("i", "j", "k"))}, body={"o": HEAT_BODY})

            def sweep_a(inner):
                inner.tasklet(ins=_stencil_body_3d("B"), outs={"o": ("A", ("i", "j", "k"))}, body={"o": HEAT_BODY})

            s.map_node(("i", "j", "k"), rng, sweep_b)
            s.map_node(("i", "j", "k"), rng, sweep_a)
    with b.state("collect") as s:
        s.library("reduce_sum", {"x": "A"}, {"y": "O"})
    return b.finish("O", ["A"])


def gemm():
    """NPBench gemm: C = 1.5 * A @ B + 1.2 * C; O = sum(C); wrt A, B, C."""
    b = ProgramBuilder(("NI", "NJ", "NK"))
    b.array("A", ("NI", "NK"), role="input", kind="real64")
    b.array("B", ("NK", "NJ"), role="input", kind="real64")
    b.array("C", ("NI", "NJ"), role="input", kind="real64")
    b.array("T", ("NI", "NJ"), kind="real64")
    b.array("T1", ("NI", "NJ"), kind="real64")
    b.array("C1", ("NI", "NJ"), kind="real64")
    b.scalar("O", role="output", kind="real64")
    with b.state("main") as s:
        s.library("matmul", {"a": "A", "b": "B"}, {"c": "T"})
        s.library("ew_unary", {"x": "T"}, {"y": "T1"}, op="scale", const=1.5)
        s.library("ew_unary", {"x": "C"}, {"y": "C1"}, op="scale", const=1.2)
        s.library("ew_binary", {"a": "T1", "b": "C1"}, {"c": "C"}, op="add")
        s.library("reduce_sum", {"x": "C"}, {"y": "O"})
    return b.finish("O", ["A", "B", "C"])


def atax():
    """NPBench atax: y = A^T (A x); O = sum(y); wrt A, x."""
    b = ProgramBuilder(("M", "N"))
    b.array("A", ("M", "N"), role="input", kind="real64")
    b.array("x", ("N", "1"), role="input", kind="real64")
    b.array("t", ("M", "1"), kind="real64")
    b.array("y", ("N", "1"), kind="real64")
    b.scalar("O", role="output", kind="real64")
    with b.state("main") as s:
        s.library("matmul", {"a": "A", "b": "x"}, {"c": "t"})
        s.library("matmul", {"a": "A", "b": "t"}, {"c": "y"}, ta=True)
        s.library("reduce_sum", {"x": "y"}, {"y": "O"})
    return b.finish("O", ["A", "x"])


def bicg():
    """NPBench bicg: s = A^T r, q = A p; O = sum(s) + sum(q); wrt A, p, r."""
    b = ProgramBuilder(("M", "N"))
    b.array("A", ("N", "M"), role="input", kind="real64")
    b.array("p", ("M", "1"), role="input", kind="real64")
    b.array("r", ("N", "1"), role="input", kind="real64")
    b.array("s", ("M", "1"), kind="real64")
    b.array("q", ("N", "1"), kind="real64")
    b.scalar("Os", kind="real64")
    b.scalar("Oq", kind="real64")
    b.scalar("O", role="output", kind="real64")
    with b.state("main") as st:
        st.library("matmul", {"a": "A", "b": "r"}, {"c": "s"}, ta=True)
        st.library("matmul", {"a": "A", "b": "p"}, {"c": "q"})
        st.library("reduce_sum", {"x": "s"}, {"y": "Os"})
        st.library("reduce_sum", {"x": "q"}, {"y": "Oq"})
        st.tasklet(ins={"a": ("Os", ()), "b": ("Oq", ())}, outs={"o": ("O", ())}, body={"o": "(add a b)"})
    return b.finish("O", ["A", "p", "r"])


def _softmax_rows(b, src, rows, cols, tag):
    """exp -> wcr rowsum map -> normalise map (the no-max form, SURVEY A)."""
    e, d, sm = f"e{tag}", f"d{tag}", f"sm{tag}"
    b.array(e, (rows, cols))
    b.array(d, (rows,))
    b.array(sm, (rows, cols))
    return e, d, sm


def softmax():
    """Row softmax over R x SM (R = NB*H*SM rows of NPBench's [NB,H,SM,SM]),
    no-max form; dependent = sum(softmax(x) * w); wrt x. real32."""
    b = ProgramBuilder(("R", "SM"))
    b.array("x", ("R", "SM"), role="input")
    b.array("w", ("R", "SM"), role="input")
    b.array("e", ("R", "SM"))
    b.array("d", ("R",))
    b.array("sm", ("R", "SM"))
    b.array("p", ("R", "SM"))
    b.scalar("O", role="output")
    with b.state("fwd") as s:
        s.library("ew_unary", {"x": "x"}, {"y": "e"}, op="exp")

        def rowsum(inner):
            inner.tasklet(ins={"v": ("e", ("r", "c"))}, outs={"o": ("d", ("r",))}, body={"o": "v"}, wcr="sum")

        s.map_node(("r", "c"), (("0", "R", "1"), ("0", "SM", "1")), rowsum)

        def norm(inner):
            inner.tasklet(ins={"v": ("e", ("r", "c")), "s": ("d", ("r",))},
                          outs={"o": ("sm", ("r", "c"))}, body={"o": "(div v s)"})

        s.map_node(("r", "c"), (("0", "R", "1"), ("0", "SM", "1")), norm)
        s.library("ew_binary", {"a": "sm", "b": "w"}, {"c": "p"}, op="mul")
        s.library("reduce_sum", {"x": "p"}, {"y": "O"})
    return b.finish("O", ["x"])


def mlp():
    """NPBench mlp: three dense layers (matmul -> bias map -> relu map), row
    softmax on the last, weighted-sum dependent; wrt x, W1..W3, b1..b3. real32."""
    b = ProgramBuilder(("NB", "C", "S0", "S1", "S2"))
    b.array("x", ("NB", "C"), role="input")
    dims = [("C", "S0"), ("S0", "S1"), ("S1", "S2")]
    for k, (i, o) in enumerate(dims, 1):
        b.array(f"W{k}", (i, o), role="input")
        b.array(f"b{k}", (o,), role="input")
        b.array(f"z{k}", ("NB", o))
        b.array(f"h{k}", ("NB", o))
        if k < 3:
            b.array(f"r{k}", ("NB", o))
    b.array("w", ("NB", "S2"), role="input")
    b.array("e", ("NB", "S2"))
    b.array("d", ("NB",))
    b.array("sm", ("NB", "S2"))
    b.array("p", ("NB", "S2"))
    b.scalar("O", role="output")
    with b.state("fwd") as s:
        src = "x"
        for k, (_, o) in enumerate(dims, 1):
            s.library("matmul", {"a": src, "b": f"W{k}"}, {"c": f"z{k}"})

            def bias(inner, k=k, o=o):
                inner.tasklet(ins={"a": (f"z{k}", ("n", "m")), "c": (f"b{k}", ("m",))},
                              outs={"o": (f"h{k}", ("n", "m"))}, body={"o": "(add a c)"})

            s.map_node(("n", "m"), (("0", "NB", "1"), ("0", o, "1")), bias)
            if k < 3:
                def relu(inner, k=k):
                    inner.tasklet(ins={"a": (f"h{k}", ("n", "m"))},
                                  outs={"o": (f"r{k}", ("n", "m"))}, body={"o": "(max a 0)"})

                s.map_node(("n", "m"), (("0", "NB", "1"), ("0", o, "1")), relu)
                src = f"r{k}"
        s.library("ew_unary", {"x": "h3"}, {"y": "e"}, op="exp")

        def rowsum(inner):
            inner.tasklet(ins={"v": ("e", ("n", "m"))}, outs={"o": ("d", ("n",))}, body={"o": "v"}, wcr="sum")

        s.map_node(("n", "m"), (("0", "NB", "1"), ("0", "S2", "1")), rowsum)

        def norm(inner):
            inner.tasklet(ins={"v": ("e", ("n", "m")), "s": ("d", ("n",))},
                          outs={"o": ("sm", ("n", "m"))}, body={"o": "(div v s)"})

        s.map_node(("n", "m"), (("0", "NB", "1"), ("0", "S2", "1")), norm)
        s.library("ew_binary", {"a": "sm", "b": "w"}, {"c": "p"}, op="mul")
        s.library("reduce_sum", {"x": "p"}, {"y": "O"})
    return b.finish("O", ["x", "W1", "W2", "W3", "b1", "b2", "b3"])


def conv2d_bias():
    """NPBench conv2d_bias, NHWC valid convolution as one 7-D wcr=sum map,
    then a bias map and a weighted-sum dependent; wrt inp, wt, bias. real32."""
    b = ProgramBuilder(("NB", "H", "W", "CI", "CO", "K"))
    b.array("inp", ("NB", "H", "W", "CI"), role="input")
    b.array("wt", ("K", "K", "CI", "CO"), role="input")
    b.array("bias", ("CO",), role="input")
    b.array("w", ("NB", "(add (sub H K) 1)", "(add (sub W K) 1)", "CO"), role="input")
    oshape = ("NB", "(add (sub H K) 1)", "(add (sub W K) 1)", "CO")
    b.array("acc", oshape)
    b.array("out", oshape)
    b.array("p", oshape)
    b.scalar("O", role="output")
    with b.state("fwd") as s:
        def conv(inner):
            inner.tasklet(
                ins={"a": ("inp", ("n", "(add i ki)", "(add j kj)", "ci")), "w": ("wt", ("ki", "kj", "ci", "co"))},
                outs={"o": ("acc", ("n", "i", "j", "co"))}, body={"o": "(mul a w)"}, wcr="sum")

        s.map_node(
            ("n", "i", "j", "co", "ki", "kj", "ci"),
            (("0", "NB", "1"), ("0", "(add (sub H K) 1)", "1"), ("0", "(add (sub W K) 1)", "1"),
             ("0", "CO", "1"), ("0", "K", "1"), ("0", "K", "1"), ("0", "CI", "1")),
            conv,
        )

        def addb(inner):
            inner.tasklet(ins={"a": ("acc", ("n", "i", "j", "co")), "c": ("bias", ("co",))},
                          outs={"o": ("out", ("n", "i", "j", "co"))}, body={"o": "(add a c)"})

        s.map_node(
            ("n", "i", "j", "co"),
            (("0", "NB", "1"), ("0", "(add (sub H K) 1)", "1"), ("0", "(add (sub W K) 1)", "1"), ("0", "CO", "1")),
            addb,
        )
        s.library("ew_binary", {"a": "out", "b": "w"}, {"c": "p"}, op="mul")
        s.library("reduce_sum", {"x": "p"}, {"y": "O"})
    return b.finish("O", ["inp", "wt", "bias"])


WORKLOADS = {
    "jacobi_2d": jacobi_2d,
    "heat_3d": heat_3d,
    "gemm": gemm,
    "atax": atax,
    "bicg": bicg,
    "softmax": softmax,
    "mlp": mlp,
    "conv2d_bias": conv2d_bias,
}
