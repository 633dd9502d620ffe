"""Device-table lowering: storage passes preserve semantics (checked on the oracle)."""

import numpy as np

import paper_1910_11141_b200 as L
from paper_1910_11141_b200 import ir
from paper_1910_11141_b200.compiler import CompiledProgram
from paper_1910_11141_b200.lowering import (demote_nonreentrant, fuse_copies, lower,
                                            recursive_functions)
from paper_1910_11141_b200.pc_vm import infer_types
from paper_1910_11141_b200.runtime import vtype_of
from conftest import load_npz, nuts_program, oracle_run


def _optimized(cp: CompiledProgram) -> CompiledProgram:
    flat, classes = demote_nonreentrant(cp.flat, dict(cp.classes), cp.labels)
    flat = fuse_copies(flat, classes)
    return CompiledProgram(flat, classes, cp.labels, cp.options, cp.stages, cp.lowering)


def test_recursive_function_detection(corpus_compiled):
    assert recursive_functions(corpus_compiled["fibonacci"][2].flat,
                               corpus_compiled["fibonacci"][2].labels) == {"fibonacci"}
    assert recursive_functions(corpus_compiled["mutual"][2].flat,
                               corpus_compiled["mutual"][2].labels) == {"pulse", "echo"}
    _, _, cp = nuts_program({"dim": 2, "rho": 0.5, "config": dict(max_depth=6, iterations=2)})
    assert recursive_functions(cp.flat, cp.labels) == {"build_tree"}


def test_nuts_demotion_removes_chain_stack():
    _, _, cp = nuts_program({"dim": 2, "rho": 0.5, "config": dict(max_depth=6, iterations=2)})
    opt = _optimized(cp)
    assert opt.classes["nuts_main.chain"] == "register"
    assert all(v.startswith("build_tree.") for v, c in opt.classes.items() if c == "stacked")
    # the chain store became an in-place vstore on the register
    vstores = [op for b in opt.flat.blocks for op in b.ops
               if not isinstance(op, ir.Pop) and op.prim.name == "vstore"]
    assert vstores and all(op.output == "nuts_main.chain" == op.inputs[0] for op in vstores)


def test_optimized_program_is_bit_identical_on_oracle(golden_meta, corpus_compiled):
    """The storage passes are pure pessimisation reversals: same bits, same traces."""
    rng = np.random.default_rng(8)
    for name, (e, _, cp) in corpus_compiled.items():
        ins = e.make_inputs(rng, 7)
        a = oracle_run(cp, ins, 64)
        b = oracle_run(_optimized(cp), ins, 64)
        assert a.output.tobytes() == b.output.tobytes(), name
        assert a.steps == b.steps, name
    meta = golden_meta["nuts"]["nuts_d2"]
    cfg, _, cp = nuts_program(meta)
    g = load_npz("nuts_runs.npz")
    ins = [np.zeros((meta["z"], 2)), g["nuts_d2_key"]]
    b = oracle_run(_optimized(cp), ins, cfg.min_stack_depth)
    assert b.output.tobytes() == g["nuts_d2_out"].tobytes()


def test_hazard_split_for_self_gradient():
    L.correlated_gaussian(3, 0.5)
    # the compiler itself routes `x = grad(x)` through a temp; a hand-written
    # flat program can still update a vector in place from a non-elementwise op
    flat = ir.parse_ir("flat\nentry 0\ninputs f.x\noutput f.x\nblock 0:\n"
                       "    update f.x = grad_g3p500 f.x\n    return\n")
    cp = CompiledProgram(flat, {"f.x": "register"}, ("f.b0",), None, {})
    types = infer_types(cp.flat, [vtype_of(np.zeros((1, 3)))])
    dp = lower(cp, types)
    names = dp.var_names
    grads = [r for r in dp.ops if r["opcode"] == 33]
    assert len(grads) == 1 and names[grads[0]["out"]].startswith("$scratch")


def test_block_tables_keep_reference_numbering():
    _, t, cp = nuts_program({"dim": 2, "rho": 0.5, "config": dict(max_depth=6, iterations=2)})
    types = infer_types(cp.flat, [vtype_of(np.zeros((1, 2))), vtype_of(np.zeros(1, np.int64))])
    dp = lower(cp, types, optimize=True)
    assert len(dp.blocks) == 41
    # block 39 (leapfrog.b2) carries both gradient invocations
    assert dp.blocks[39]["grads"] == 2 and dp.blocks["grads"].sum() == 2
    for bi, blk in enumerate(cp.flat.blocks):
        t_ = blk.terminator
        if isinstance(t_, ir.PushJump):
            assert (dp.blocks[bi]["a"], dp.blocks[bi]["b"]) == (t_.jump_to, t_.return_to)


def _sim_matches_oracle(cp, ins, depth, opt):
    from oracle import table_sim

    types = infer_types(cp.flat, [vtype_of(a) for a in ins])
    dp = lower(cp, types, optimize=opt)
    out, traces = table_sim.run(dp, ins, depth)
    ref = oracle_run(cp, ins, depth, lane_traces=True)
    want = ref.output.astype(np.uint64) if ref.output.dtype == np.bool_ else ref.output
    want = np.ascontiguousarray(want).view(np.uint64).reshape(out.shape)
    if ref.output.dtype.kind == "f":
        np.testing.assert_allclose(out.view(np.float64), want.view(np.float64), rtol=1e-12, atol=1e-15)
    else:
        assert np.array_equal(out, want)
    assert all(a == b for a, b in zip(traces, ref.lane_blocks))
    return dp


def test_device_tables_simulate_to_oracle_results(corpus_compiled):
    """Storage assignment (arena, views, in-place vcat, demotion) preserves every lane's result."""
    import itertools

    from paper_1910_11141_b200.compiler import CompileOptions

    rng = np.random.default_rng(3)
    for name, (e, cfg, _) in corpus_compiled.items():
        for bits in itertools.product([True, False], repeat=4):
            cp = L.compile_program(cfg, CompileOptions(*bits))
            ins = e.make_inputs(rng, 3)
            for opt in (False, True):
                _sim_matches_oracle(cp, ins, 64, opt)


def test_nuts_tables_shrink_and_stay_exact():
    cfg, t, cp = nuts_program({"dim": 100, "rho": 0.5, "config": dict(max_depth=10, iterations=3)})
    ins = [np.zeros((2, 100)), np.array([5, 6], np.int64)]
    plain = _sim_matches_oracle(cp, ins, cfg.min_stack_depth, False)
    opt = _sim_matches_oracle(cp, ins, cfg.min_stack_depth, True)
    assert opt.flat_rows * 5 < plain.flat_rows


def test_nuts_fusions_fire():
    """The fused momentum draw and the dead-save pass apply to NUTS-lite at every
    dimension (odd dims leave the last pair's sine unused)."""
    from paper_1910_11141_b200.lowering import OPCODES

    for dim in (2, 5, 100):
        cfg, t, cp = nuts_program({"dim": dim, "rho": 0.5, "config": dict(max_depth=4, iterations=2)})
        types = infer_types(cp.flat, [vtype_of(np.zeros((1, dim))), vtype_of(np.zeros(1, np.int64))])
        dp = lower(cp, types, optimize=True)
        codes = set(dp.ops["opcode"].tolist())
        assert OPCODES["normals"] in codes and OPCODES["alloc"] in codes, dim
        nrm = dp.ops[dp.ops["opcode"] == OPCODES["normals"]][0]
        assert (nrm["imm0"], nrm["imm1"]) == (dim, (dim + 1) // 2)
        plain = lower(cp, types, optimize=False)
        assert OPCODES["normals"] not in set(plain.ops["opcode"].tolist())


def test_superblock_forwarding_and_fused_leaf_logpdf():
    """With superblocks the leapfrog reads its arguments from the caller's sources (the call
    block's argument copies disappear), writes back nothing the program never reads, and
    fills the register the leaf's logpdf reads in fast mode."""
    from paper_1910_11141_b200.lowering import OPCODES

    cfg, t, cp = nuts_program({"dim": 100, "rho": 0.5, "config": dict(max_depth=6, iterations=2)})
    types = infer_types(cp.flat, [vtype_of(np.zeros((1, 100))), vtype_of(np.zeros(1, np.int64))])
    dp = lower(cp, types, optimize=True, superblocks=True)
    (lf,) = dp.ops[dp.ops["opcode"] == OPCODES["leapfrog"]]
    names = [dp.var_names[int(v)] for v in lf["in"][:2]]
    assert names == ["build_tree.q", "build_tree.p"]  # forwarded from the caller
    assert int(lf["kind"]) & 1 == 0  # q, p are dead after the return: no write-back
    assert int(lf["bits"]) == -1  # g and i are dead too
    lp_var = (int(lf["kind"]) >> 1) - 1
    assert dp.var_names[lp_var] == "leapfrog.$lp"
    cached = dp.ops[(dp.ops["opcode"] == OPCODES["logpdf"]) & (dp.ops["bits"] > 0)]
    assert len(cached) == 1 and int(cached[0]["bits"]) - 1 == lp_var
    # the call block (build_tree.b1) no longer copies vectors into leapfrog.q / leapfrog.p
    call = dp.blocks[cp.labels.index("build_tree.b1")]
    ops = dp.ops[call["op_begin"]:call["op_begin"] + call["op_count"]]
    assert not any(dp.var_names[int(o["out"])] in ("leapfrog.q", "leapfrog.p") for o in ops)
