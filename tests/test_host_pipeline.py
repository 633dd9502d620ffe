"""Host pipeline (frontend + compiler + IR text) reproduces the reference exactly.

The golden IR texts were printed by the reference compiler (tests/golden/
make_golden.py). Block numbering and storage classes must match, because the
device VM runs exactly this flat program and pc traces are block indices.
Mirrors reference tests test_compiler.py / test_ir.py / test_frontend.py.
"""

import itertools

import numpy as np
import pytest

import paper_1910_11141_b200 as L
from paper_1910_11141_b200 import ir
from paper_1910_11141_b200.compiler import CompileOptions, cancel_pop_push, flatten
from paper_1910_11141_b200.errors import LoweringError, ParseError, TypeInferenceError
from paper_1910_11141_b200.pc_vm import infer_types
from paper_1910_11141_b200.runtime import VType
from conftest import nuts_program

ALL_OPTIONS = [CompileOptions(*bits) for bits in itertools.product([True, False], repeat=4)]


def test_corpus_ir_matches_reference(golden_meta, corpus_compiled):
    for name, meta in golden_meta["corpus"].items():
        _, _, cp = corpus_compiled[name]
        assert ir.print_ir(cp.flat) == meta["ir"], name
        assert cp.classes == meta["classes"], name


def test_nuts_ir_matches_reference(golden_meta):
    for name, meta in golden_meta["nuts"].items():
        _, _, cp = nuts_program(meta)
        assert ir.print_ir(cp.flat) == meta["ir"], name


def test_nuts_source_shape():
    t = L.correlated_gaussian(2, 0.5)
    src = L.nuts_lite_source(L.NutsConfig(step_size=0.125), t)
    assert "0.125" in src and "grad_g2p500" in src and "logpdf_g2p500" in src
    assert L.nuts_lite_source(L.workloads.TINY_NUTS) == L.nuts_lite_source(L.workloads.TINY_NUTS, t)


def test_nuts_flat_program_has_41_blocks():
    cfg, t, cp = nuts_program({"dim": 2, "rho": 0.5, "config": dict(max_depth=10, iterations=3)})
    assert len(cp.flat.blocks) == 41 and cp.flat.halt_index == 41
    assert {"leapfrog.q", "leapfrog.p"} <= cp.registers
    assert "nuts_main.chain" in cp.stacked


@pytest.mark.parametrize("opts", ALL_OPTIONS, ids=str)
def test_all_pass_subsets_compile_and_validate(corpus_compiled, opts):
    for name, (_, cfg, _) in corpus_compiled.items():
        cp = L.compile_program(cfg, opts)
        assert ir.validate_flat(cp.flat, cp.stacked) == []


def test_print_parse_round_trip(corpus_compiled):
    for name, (_, cfg, cp) in corpus_compiled.items():
        assert ir.parse_ir(ir.print_ir(cp.flat)) == cp.flat
        assert ir.parse_ir(ir.print_ir(cfg)) == cfg


def test_cancellation_idempotent(corpus_compiled):
    for _, cfg, _ in corpus_compiled.values():
        flat, _ = flatten(cfg)
        once = cancel_pop_push(flat)
        assert cancel_pop_push(once) == once


def test_fib_stacked_set(corpus_compiled):
    assert corpus_compiled["fibonacci"][2].stacked == {"fibonacci.n", "fibonacci.left", "fibonacci._ret"}


def test_loop_programs_are_stack_free(corpus_compiled):
    for name in ("countdown", "twosite", "poly"):
        assert corpus_compiled[name][2].stacked == frozenset()


def test_frontend_errors():
    with pytest.raises(ParseError):
        L.parse_source("def f(x) { return x }")
    with pytest.raises(LoweringError):
        L.compile_source("def f(x) { return y; }")
    with pytest.raises(LoweringError):
        L.compile_source("def f(x) { _t0 = x; return x; }")
    with pytest.raises(LoweringError):
        L.compile_source("def sqrt(x) { return x; }")
    with pytest.raises(LoweringError):
        L.compile_source("def f(x) { return g(x); }")


def test_type_inference_rules(corpus_compiled):
    cp = corpus_compiled["fibonacci"][2]
    types = infer_types(cp.flat, [VType("i64")])
    assert types["fibonacci.n"] == VType("i64")
    with pytest.raises(TypeInferenceError):
        infer_types(cp.flat, [VType("i64"), VType("i64")])
    bad = L.compile_program(L.compile_source("def f(x) { v = vfill:2(x); v = vfill:3(x); return vget(v, 0); }"))
    with pytest.raises(TypeInferenceError, match="f.v"):
        infer_types(bad.flat, [VType("f64")])
    nb = L.compile_program(L.compile_source("def f(x) { while (x) { x = x - 1; } return x; }"))
    with pytest.raises(TypeInferenceError, match="bool"):
        infer_types(nb.flat, [VType("i64")])


def test_nuts_config_validation():
    c = L.NutsConfig()
    assert (c.step_size, c.leaf_steps, c.max_depth, c.iterations) == (0.25, 4, 6, 400)
    assert L.NutsConfig(max_depth=6).min_stack_depth == 10
    for kw in ({"leaf_steps": 0}, {"max_depth": 0}, {"iterations": 0}, {"step_size": 0.0}):
        with pytest.raises(ValueError):
            L.NutsConfig(**kw)


def test_target_registry_and_names():
    assert L.correlated_gaussian(2, 0.5) is L.correlated_gaussian(2, 0.5)
    assert L.correlated_gaussian(3, -0.2).name == "g3m200"
    assert L.logistic_regression(40, 3, seed=9).name == "lr40x3s9"
    with pytest.raises(ValueError):
        L.correlated_gaussian(2, 1.0)
    with pytest.raises(ValueError):
        L.correlated_gaussian(3, -0.6)
    t = L.correlated_gaussian(1000, 9999 / 10999)
    assert t.name == "g1000p909"
    assert abs(np.linalg.cond(t.cov) - 1e4) < 1e-3


def test_metrics_json_round_trip():
    tr = L.ScheduleTrace(engine="pc", z=4)
    tr.record("f.b0", 3, {"add": 2, "grad_x": 1})
    tr.record("f.b1", 1, {"grad_x": 2})
    tr.record_stack_op("f.n", "push")
    back = L.metrics.trace_from_json(L.metrics.trace_to_json(tr))
    assert back.steps == tr.steps and back.stack_ops == tr.stack_ops
    assert L.utilization(tr, {"grad_x"}) == pytest.approx((3 + 2) / (4 * 3))
    assert L.trace_to_csv(tr).splitlines()[1] == "0,f.b0,3"
