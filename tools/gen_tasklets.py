"""Ahead-of-time tasklet bodies for gfb_map2 (writes csrc/gen_tasklets.cu).

The engine's vectorised map kernels (csrc/map2_kernels.cuh) take the tasklet
body as a policy type. At run time gfb_map2_launch hashes the descriptor's
bytecode (m2_key in csrc/map2.cu) and, when a body compiled here matches,
runs that instantiation instead of the register-stack bytecode evaluator, so
the per-point work is the tasklet's arithmetic and nothing else.

Which bodies: every pointwise map / single-dimension reduction the host
lowering produces for the bundled programs (paper_2509_02197_b200/programs:
the BASELINE.json workloads at their config and small sizes, the reference
corpus programs at their golden-case sizes, and the bundled checkpoint
plans). Anything else still runs, on the evaluator.

    python tools/gen_tasklets.py            # (re)write csrc/gen_tasklets.cu
    python tools/gen_tasklets.py --check    # exit 1 if the file is stale
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2509_02197_b200 import _lib as L  # noqa: E402
from paper_2509_02197_b200 import workloads as W  # noqa: E402
from paper_2509_02197_b200.api import lower_gradient  # noqa: E402
from paper_2509_02197_b200.lowering import Map2Op  # noqa: E402

OUT = os.path.join(REPO, "paper_2509_02197_b200", "csrc", "gen_tasklets.cu")
GOLD = os.path.join(REPO, "tests", "golden")

BIN = {L.OP_ADD: "GFB_OP_ADD", L.OP_SUB: "GFB_OP_SUB", L.OP_MUL: "GFB_OP_MUL", L.OP_DIV: "GFB_OP_DIV",
       L.OP_IDIV: "GFB_OP_IDIV", L.OP_MOD: "GFB_OP_MOD", L.OP_MIN: "GFB_OP_MIN", L.OP_MAX: "GFB_OP_MAX",
       L.OP_POW: "GFB_OP_POW"}
UN = {L.OP_NEG: "GFB_OP_NEG", L.OP_SIN: "GFB_OP_SIN", L.OP_COS: "GFB_OP_COS", L.OP_EXP: "GFB_OP_EXP",
      L.OP_LOG: "GFB_OP_LOG", L.OP_SQRT: "GFB_OP_SQRT", L.OP_TANH: "GFB_OP_TANH", L.OP_ABS: "GFB_OP_ABS",
      L.OP_SIGN: "GFB_OP_SIGN"}


def m2_key(mode, f64, n_in, segs, words, umask=0) -> int:
    """FNV-1a, byte-identical to gfb::m2_key (csrc/map2.cu)."""
    h = 1469598103934665603
    mask = (1 << 64) - 1

    def mix(x):
        nonlocal h
        x &= 0xFFFFFFFF
        for b in range(4):
            h ^= (x >> (8 * b)) & 0xFF
            h = (h * 1099511628211) & mask

    mix(mode)
    mix(f64)
    mix(n_in)
    mix(len(segs))
    for start, n in segs:
        mix(start)
        mix(n)
        for pc in range(start, start + n):
            mix(words[pc])
    if umask:
        mix(0x55000000 | umask)
    return h


def uniform_mask(op: Map2Op) -> int:
    """Inputs constant along the innermost loop dimension (gfb::m2_uniform_mask)."""
    if op.compute_f64 or not op.ext:
        return 0
    m = 0
    for k, (_b, _c0, st) in enumerate(op.ins[:32]):
        if int(st[len(op.ext) - 1]) == 0:
            m |= 1 << k
    return m


def signature(op: Map2Op):
    f64 = 1 if op.compute_f64 else 0
    return (op.mode, f64, len(op.ins), tuple(op.segs), tuple(op.code_words[:max(s + n for s, n in op.segs)]),
            uniform_mask(op))


def collect():
    sigs = {}

    def take(low):
        for op in low.ops:
            if isinstance(op, Map2Op):
                sigs.setdefault(signature(op), None)

    for cfg, (name, params) in W.CONFIGS.items():
        prog, bundle = W.load(name)
        take(lower_gradient(prog, bundle, params, W.input_shapes(prog, params)).low)
    for name, plist in W.SMALL_PARAMS.items():
        prog, bundle = W.load(name)
        for params in plist:
            take(lower_gradient(prog, bundle, params, W.input_shapes(prog, params)).low)
    idx_path = os.path.join(GOLD, "index.json")
    if os.path.exists(idx_path):
        idx = json.load(open(idx_path))
        from paper_2509_02197_b200.api import load_plan

        for cid, meta in list(idx.get("cases", {}).items()) + list(idx.get("examples", {}).items()):
            try:
                prog, bundle = W.load(meta["workload"])
                take(lower_gradient(prog, bundle, meta["params"], W.input_shapes(prog, meta["params"])).low)
            except Exception:  # unsupported constructs stay on their own paths
                pass
        for cid, meta in idx.get("plans", {}).items():
            try:
                pb = load_plan(os.path.join(GOLD, "plans", cid))
                take(lower_gradient(pb.forward, None, meta["params"], W.input_shapes(pb.forward, meta["params"]),
                                    plan=pb).low)
            except Exception:
                pass
    # the config-scale checkpoint plans (recompute fused into the adjoint maps)
    pidx = os.path.join(W.PROG_DIR, "plans", "index.json")
    if os.path.exists(pidx):
        from paper_2509_02197_b200.api import load_plan

        for cid, meta in json.load(open(pidx)).items():
            pb = load_plan(os.path.join(W.PROG_DIR, "plans", cid))
            take(lower_gradient(pb.forward, None, meta["params"], W.input_shapes(pb.forward, meta["params"]),
                                plan=pb).low)
    return sorted(sigs)


def body_code(words, segs, umask=0) -> str:
    """Straight-line body of each output's stack code. With a uniform mask
    (row-scalar inputs) stack slots computed only from uniform inputs and
    constants stay one-element arrays (u*): evaluated once per lane, broadcast
    when they meet a per-point slot (s*)."""
    lines = []
    for o, (start, n) in enumerate(segs):
        stack, stmts, maxd, maxu = [], [], 0, 0

        def push(scalar):
            nonlocal maxd, maxu
            depth = len(stack)
            name = f"u{depth}" if scalar else f"s{depth}"
            stack.append((name, scalar))
            if scalar:
                maxu = max(maxu, depth + 1)
            else:
                maxd = max(maxd, depth + 1)
            return name

        def as_vec(slot, depth):
            name, scalar = slot
            if not scalar:
                return name
            vec = f"s{depth}"
            stmts.append(f"m2_fill<T, V>({vec}, {name}[0]);")
            return vec

        for pc in range(start, start + n):
            w = words[pc]
            op, arg = w & 63, w >> 10
            if op == L.OP_IN:
                if (umask >> arg) & 1:
                    nm = push(True)
                    stmts.append(f"{{ T t_[V]; fetch({arg}, t_); {nm}[0] = t_[0]; }}")
                else:
                    nm = push(False)
                    stmts.append(f"fetch({arg}, {nm});")
            elif op == L.OP_CONST:
                nm = push(bool(umask))
                if umask:
                    stmts.append(f"{nm}[0] = (T)d.consts[{arg}];")
                else:
                    stmts.append(f"m2_fill<T, V>({nm}, (T)d.consts[{arg}]);")
            elif op in UN:
                name, scalar = stack[-1]
                if scalar:
                    stmts.append(f"m2_unary<T, 1>({UN[op]}, {name}, vm ? 1u : 0u, bad);")
                else:
                    stmts.append(f"m2_unary<T, V>({UN[op]}, {name}, vm, bad);")
            else:
                b = stack.pop()
                a = stack.pop()
                depth = len(stack)
                if a[1] and b[1]:
                    nm = push(True)
                    if a[0] != nm:
                        stmts.append(f"{nm}[0] = {a[0]}[0];")
                    stmts.append(f"m2_binary<T, 1>({BIN[op]}, {nm}, {b[0]}, vm ? 1u : 0u, bad);")
                elif op == L.OP_DIV and b[1] and not a[1]:
                    # a vector over a per-lane scalar (a row value): one
                    # reciprocal per lane, then products (<= 1.5 ulp from
                    # the correctly rounded quotient; zero still raises)
                    if a[0] != f"s{depth}":
                        stmts.append(f"m2_copy<T, V>(s{depth}, {a[0]});")
                    maxd = max(maxd, depth + 1)
                    stmts.append(f"m2_div_scalar<T, V>(s{depth}, {b[0]}[0], vm, bad);")
                    stack.append((f"s{depth}", False))
                else:
                    # destination slot s{depth}; the right operand goes to s{depth + 1}
                    bv = as_vec(b, depth + 1) if b[1] else b[0]
                    if a[1]:
                        stmts.append(f"m2_fill<T, V>(s{depth}, {a[0]}[0]);")
                    elif a[0] != f"s{depth}":
                        stmts.append(f"m2_copy<T, V>(s{depth}, {a[0]});")
                    maxd = max(maxd, depth + 2)
                    stmts.append(f"m2_binary<T, V>({BIN[op]}, s{depth}, {bv}, vm, bad);")
                    stack.append((f"s{depth}", False))
        res, rs = stack[-1]
        decl = []
        if maxd:
            decl.append("T " + ", ".join(f"s{i}[V]" for i in range(maxd)) + ";")
        if maxu:
            decl.append("T " + ", ".join(f"u{i}[1]" for i in range(maxu)) + ";")
        tail = f"m2_fill<T, V>(r, {res}[0]);" if rs else f"m2_copy<T, V>(r, {res});"
        body = " ".join(decl + stmts + [tail])
        lines.append(f"    {'if' if o == 0 else 'else if'} (o == {o}) {{ {body} }}")
    return "\n".join(lines)


def generate() -> str:
    sigs = collect()
    out = [
        "// GENERATED by tools/gen_tasklets.py -- do not edit.",
        "// Ahead-of-time tasklet bodies of the bundled programs for gfb_map2",
        "// (see the generator's docstring and csrc/map2_kernels.cuh).",
        '#include "map2_kernels.cuh"',
        "",
        "namespace gfb {",
        "",
        "template <typename T, int V>",
        "__device__ __forceinline__ void m2_fill(T (&x)[V], T c) {",
        "#pragma unroll",
        "  for (int v = 0; v < V; ++v) x[v] = c;",
        "}",
        "template <typename T, int V>",
        "__device__ __forceinline__ void m2_copy(T (&x)[V], const T (&y)[V]) {",
        "#pragma unroll",
        "  for (int v = 0; v < V; ++v) x[v] = y[v];",
        "}",
        "template <typename T, int V>",
        "__device__ __forceinline__ void m2_div_scalar(T (&x)[V], T c, uint32_t vm, uint32_t &bad) {",
        "  if (vm && c == T(0)) bad |= GFB_EBIT_DIV0;",
        "  const T rc = T(1) / c;",
        "#pragma unroll",
        "  for (int v = 0; v < V; ++v) x[v] = x[v] * rc;",
        "}",
        "",
    ]
    table = []
    for i, (mode, f64, n_in, segs, words, umask) in enumerate(sigs):
        key = m2_key(mode, f64, n_in, segs, words, umask)
        T, V = ("double", 2) if f64 else ("float", 4)
        out += [
            f"struct GenBody{i} {{  // mode {mode}, {'fp64' if f64 else 'fp32'}, {n_in} inputs, {len(segs)} outputs"
            + (f", row-scalar inputs 0x{umask:x}" if umask else ""),
            f"  static constexpr int kNIn = {n_in}, kNOut = {len(segs)};",
            f"  static constexpr uint32_t kRowScalar = 0x{umask:x}u;  // inputs with stride 0 along the row",
            "  template <typename T, int V, typename F>",
            "  static __device__ __forceinline__ void eval(const gfb_map2_desc &d, int o, F &fetch, uint32_t vm,",
            "                                              T (&r)[V]) {",
            "    uint32_t bad = 0;",
            body_code(words, segs, umask),
            "    if (bad) raise_bits(d.err, bad);",
            "  }",
            "};",
            f"static int gen_launch{i}(const gfb_map2_desc &d, cudaStream_t st) {{",
            f"  return launch_map2<{T}, {V}, GenBody{i}, {mode}{', true' if umask else ''}>(d, st);",
            "}",
            "",
        ]
        table.append(f"    {{0x{key:016x}ull, gen_launch{i}}},")
    out += ["struct M2Special {", "  uint64_t key;", "  int (*launch)(const gfb_map2_desc &, cudaStream_t);", "};",
            "extern const M2Special kM2Specials[];", "extern const int kM2NumSpecials;",
            "const M2Special kM2Specials[] = {"] + (table or ["    {0ull, nullptr},"]) + [
            "};", f"const int kM2NumSpecials = {len(table)};", "", "}  // namespace gfb", ""]
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    text = generate()
    old = open(OUT).read() if os.path.exists(OUT) else None
    if args.check:
        sys.exit(0 if old == text else 1)
    if old != text:
        with open(OUT, "w") as f:
            f.write(text)
    print(f"{OUT}: {text.count('struct GenBody')} bodies")


if __name__ == "__main__":
    main()
