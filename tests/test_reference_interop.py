"""Programs compiled by the reference `lockstep` compiler are accepted by this engine.

Runs only where the reference package is importable (the builder container); the
conversion itself is pure host code, so the check needs no GPU: it compares the
adopted flat program with this package's own compilation.
"""

import sys

import pytest

import paper_1910_11141_b200 as L
from paper_1910_11141_b200 import ir
from paper_1910_11141_b200.compiler import adopt

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def lockstep():
    sys.path.insert(0, REF)
    try:
        import lockstep as R
    except ImportError:
        pytest.skip("reference package not present (GPU box)")
    finally:
        sys.path.remove(REF)
    return R


def test_adopt_reference_compiled_programs(lockstep):
    L.corpus()  # registers this package's targets (the corpus includes NUTS-lite)
    for e in lockstep.corpus():
        ref_cp = lockstep.compile_program(lockstep.compile_source(e.source, e.entry))
        mine = L.compile_program(L.compile_source(e.source, e.entry))
        got = adopt(ref_cp)
        assert got.flat == mine.flat and got.classes == mine.classes and got.labels == mine.labels
        assert ir.print_ir(got.flat) == ir.print_ir(mine.flat)
