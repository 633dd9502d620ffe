"""The host pipeline is the reference's own, and the device reads its targets exactly.

The package re-exports the reference `lockstep` front end, compiler, IR types,
generator, traces and exceptions unchanged (paper_1910_11141_b200/reference.py);
the engine consumes the reference's `CompiledProgram`. These checks pin that
(the installed reference compiles the goldens it minted, tests/golden) and that
`workloads.device_target` reads the very parameter arrays the reference's own
kernels compute with (closure cells).
"""

import numpy as np

import paper_1910_11141_b200 as L
from paper_1910_11141_b200 import ir
from paper_1910_11141_b200.reference import lockstep as R
from conftest import load_npz, nuts_program


def test_pipeline_is_the_reference():
    assert L.compile_source is R.compile_source and L.compile_program is R.compile_program
    assert L.nuts_lite_source is R.nuts_lite_source and L.NutsConfig is R.NutsConfig
    assert L.StackOverflow is R.StackOverflow and L.ScheduleTrace is R.ScheduleTrace
    assert ir.FlatProgram is R.ir.FlatProgram and ir.PushJump is R.ir.PushJump
    assert L.infer_types is R.pc_vm.infer_types


def test_installed_reference_compiles_the_pinned_goldens(golden_meta, corpus_compiled):
    for name, meta in golden_meta["corpus"].items():
        _, _, cp = corpus_compiled[name]
        assert ir.print_ir(cp.flat) == meta["ir"], name
        assert cp.classes == meta["classes"], name
    for name, meta in golden_meta["nuts"].items():
        _, _, cp = nuts_program(meta)
        assert ir.print_ir(cp.flat) == meta["ir"], name


def test_device_targets_read_the_reference_parameters():
    e = load_npz("gauss_logpdf.npz")
    for d in (2, 5, 25, 100, 128):
        t = L.correlated_gaussian(d, 0.5)
        dt = L.device_target(t.name)
        assert dt.kind == 1 and dt.dim == d and dt.grad == t.grad and dt.logpdf == t.logpdf
        assert np.array_equal(dt.params["prec"], e[f"P{d}"])
        zero = np.zeros((1, d))
        assert dt.params["norm"] == R.runtime.resolve_kernel(t.logpdf).fn((zero,), 1)[0]
        assert dt.grad_flops == 2 * d * d
    from oracle import lockstep_oracle as O

    g = load_npz("logreg.npz")
    for n, d, seed in ((25, 3, 2), (200, 5, 7), (1000, 25, 0)):
        t = L.logistic_regression(n, d, seed)
        dt = L.device_target(t.name)
        assert dt.kind == 2 and dt.params["sx"].shape == (n, d) and dt.grad_flops == 4 * n * d
        w = g[f"lr{n}x{d}s{seed}_w"]
        assert O.logreg_grad(w, dt.params["sx"]).tobytes() == g[f"lr{n}x{d}s{seed}_g"].tobytes()


def test_targets_without_parameters_have_no_device_form():
    R.runtime.register_kernel("grad_custom_host_only", 1, lambda ins, z: -ins[0],
                              lambda ins: ins[0])
    assert L.runtime.device_op("grad_custom_host_only") is None
    assert L.runtime.device_op("logpdf_no_such_target") is None
    assert L.runtime.device_op("add").opcode == L.runtime.OPCODES["add"]
    assert L.runtime.device_op("vslice:3:7").imm1 == 7
