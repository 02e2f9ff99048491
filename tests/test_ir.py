"""Host-side IR logic against the reference: JSON wire format, schedule
order and write-version numbering (the pieces the engine re-implements)."""
import json
import os
import sys

import pytest

from conftest import REF_SRC
from paper_2509_02197_b200 import workloads as W
from paper_2509_02197_b200.ir import (
    State,
    dump_program,
    load_program,
    number_writes,
    parse_sexpr,
    schedule,
    to_sexpr,
    walk_blocks,
)

PROGRAMS = sorted(f[:-9] for f in os.listdir(W.PROG_DIR) if f.endswith(".fwd.json"))


@pytest.mark.parametrize("name", PROGRAMS)
def test_wire_roundtrip_is_idempotent(name):
    for suffix in (".fwd.json", ".bwd.json"):
        path = os.path.join(W.PROG_DIR, name + suffix)
        p = load_program(path)
        text = dump_program(p)
        assert dump_program(load_program(text)) == text


def test_sexpr_roundtrip():
    for s in ["(add (mul N N) 3)", "(mul 0.2 (add cc ww))", "(idiv (sub i 1) 2)", "(neg (sin x))", "-3", "2.5"]:
        assert to_sexpr(parse_sexpr(s)) == s


@pytest.mark.ref
@pytest.mark.parametrize("name", PROGRAMS)
def test_schedule_and_versions_match_reference(name):
    sys.path.insert(0, REF_SRC)
    from gradflow.frontend import load_program as ref_load
    from gradflow.ir import schedule as ref_schedule
    from gradflow.ir import walk_blocks as ref_walk
    from gradflow.versions import analyze_versions

    for suffix in (".fwd.json", ".bwd.json"):
        path = os.path.join(W.PROG_DIR, name + suffix)
        mine, ref = load_program(path), ref_load(path)
        for (_, a), (_, b) in zip(walk_blocks(mine.region), ref_walk(ref.region), strict=True):
            if isinstance(a, State):
                assert schedule(a.graph) == ref_schedule(b.graph)
        vo, lo = number_writes(mine)
        info = analyze_versions(ref)
        assert vo == info.write_version
        assert lo == info.write_loops


@pytest.mark.ref
def test_reference_serializer_reads_our_output():
    sys.path.insert(0, REF_SRC)
    from gradflow.frontend import parse_program, serialize_program

    for name in PROGRAMS:
        p = load_program(os.path.join(W.PROG_DIR, name + ".bwd.json"))
        ref = parse_program(dump_program(p))
        assert json.loads(serialize_program(ref)) == json.loads(
            open(os.path.join(W.PROG_DIR, name + ".bwd.json")).read())
