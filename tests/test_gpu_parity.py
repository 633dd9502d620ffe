"""Parity of the B200 VM with the reference, through the C ABI (needs a GPU).

Mirrors the reference suites test_pc_vm.py and test_acceptance.py. Integer
and control results (outputs of integer programs, global step traces,
per-lane program-counter traces, stack-op counts, fault reports, rng) must
be bit-exact; float chain positions agree within the tolerance stated per
test (the reference gradient goes through OpenBLAS, which is not
reproducible even across its own batch widths — SURVEY.md §0.4).
"""

import itertools

import numpy as np
import pytest

import paper_1910_11141_b200 as L
from paper_1910_11141_b200 import _native, pc_vm
from paper_1910_11141_b200.compiler import CompileOptions
from paper_1910_11141_b200.errors import StackOverflow, StepLimitExceeded
from conftest import load_npz, nuts_program, oracle_run, split_lanes

pytestmark = pytest.mark.gpu

Z_CYCLE = (1, 2, 4, 7, 32)
ALL_OPTIONS = [CompileOptions(*bits) for bits in itertools.product([True, False], repeat=4)]
SPIN = "def spin(n) { while (0 <= n) { n = n + 1; } return n; }"
# float tolerance for whole chains (many leapfrog steps); per-step is 1e-12 below
CHAIN_RTOL = 1e-9


def assert_matches(got, ref, label, rtol=1e-12):
    if got.dtype.kind in "ib":
        assert np.array_equal(got, ref), label
    else:
        np.testing.assert_allclose(got, ref, rtol=rtol, atol=0.0, err_msg=label)


def test_device_present():
    assert _native.device_count() >= 1


def test_corpus_golden_runs(golden_meta, corpus_compiled):
    g = load_npz("corpus_runs.npz")
    for name, meta in golden_meta["corpus"].items():
        _, _, cp = corpus_compiled[name]
        for run in meta["runs"]:
            ins = [g[f"{run['tag']}_in{k}"] for k in range(run["n_inputs"])]
            out, tr = L.run(cp, ins, depth=64)
            want = g[f"{run['tag']}_out"]
            assert_matches(out, want, run["tag"])
            assert [[s.block, s.active] for s in tr.steps] == run["steps"], run["tag"]
            assert tr.stack_ops == run["stack_ops"], run["tag"]


def test_fifty_random_batches_per_program(corpus_compiled):
    """TestOracleEquivalence (reference test_acceptance.py:54-74) against the oracle."""
    rng = np.random.default_rng(2024)
    for name, (e, cfg, _) in corpus_compiled.items():
        variants = {}
        for b in range(50 if name != "nuts_lite" else 15):
            z = Z_CYCLE[b % len(Z_CYCLE)]
            ins = e.make_inputs(rng, z)
            opts = ALL_OPTIONS[b % len(ALL_OPTIONS)]
            if opts not in variants:
                variants[opts] = L.compile_program(cfg, opts)
            ref = oracle_run(variants[opts], ins, 64).output
            got, _ = L.run(variants[opts], ins, depth=64)
            assert_matches(got, ref, f"{name} batch {b}")


def test_all_sixteen_pass_subsets_bit_identical(corpus_compiled):
    rng = np.random.default_rng(5)
    for name, (e, cfg, _) in corpus_compiled.items():
        ins = e.make_inputs(rng, 4)
        outs = {L.run(L.compile_program(cfg, o), ins, depth=64)[0].tobytes() for o in ALL_OPTIONS}
        assert len(outs) == 1, name


@pytest.mark.parametrize("ins,want", [([3, 7, 4, 5], [3, 21, 5, 8]), ([6, 7, 8, 9], [13, 21, 34, 55])])
def test_fib_goldens(corpus_compiled, ins, want):
    out, tr = L.run(corpus_compiled["fibonacci"][2], [np.array(ins)], depth=32)
    assert out.tolist() == want
    assert tr.engine == "pc" and tr.z == 4


@pytest.mark.parametrize("k,want", [(4, 45), (6, 123), (8, 327)])
def test_cross_depth_frozen_step_counts(corpus_compiled, k, want):
    """Frozen pc step counts of reference test_acceptance.py:106-129, plus depth mixing."""
    mixed = []

    def observer(m, b, sel):
        ptr = m.stacks["fibonacci.n"].pointers
        mixed.append(len(np.unique(ptr[sel])) > 1)

    _, tr = L.run(corpus_compiled["fibonacci"][2], [np.array([k, k + 1])], depth=48, observer=observer)
    assert tr.step_count == want
    assert any(mixed)
    _, fast = L.run(corpus_compiled["fibonacci"][2], [np.array([k, k + 1])], depth=48)
    assert fast.step_count == want


def test_loop_programs_touch_no_data_stack(corpus_compiled):
    for name, args in (("countdown", [7]), ("poly", [3]), ("twosite", [9])):
        _, tr = L.run(corpus_compiled[name][2], [np.array(args)], depth=16)
        assert tr.stack_ops == {}


def test_stack_traffic_and_balance(corpus_compiled):
    _, tr = L.run(corpus_compiled["fibonacci"][2], [np.array([8, 3, 6])], depth=32)
    assert set(tr.stack_ops) == {"fibonacci.n", "fibonacci.left", "fibonacci._ret"}
    for var, ops in tr.stack_ops.items():
        assert ops["push"] == ops["pop"], var


def test_overflow_names_lane_variable_and_block(corpus_compiled):
    fib = corpus_compiled["fibonacci"][2]
    with pytest.raises(StackOverflow) as ei:
        L.run(fib, [np.array([10])], depth=3)
    err = ei.value
    assert err.lane == 0 and err.variable.startswith("fibonacci.")
    assert err.block is not None and err.block.startswith("fibonacci.")
    assert "stack overflow" in str(err) and "lane 0" in str(err)
    with pytest.raises(StackOverflow) as ei:
        L.run(fib, [np.array([1, 10, 1])], depth=3)
    assert ei.value.lane == 1
    with pytest.raises(StackOverflow):
        L.run(fib, [np.array([10])], depth=2)


def test_fault_report_matches_oracle(corpus_compiled):
    from oracle.lockstep_oracle import OracleFault

    fib = corpus_compiled["fibonacci"][2]
    for ins in ([np.array([10])], [np.array([1, 10, 1])], [np.array([9, 10, 3, 12])]):
        with pytest.raises(OracleFault) as want:
            oracle_run(fib, ins, 3)
        with pytest.raises(StackOverflow) as got:
            L.run(fib, ins, depth=3)
        assert (got.value.variable, got.value.lane, got.value.block) == \
            (want.value.variable, want.value.lane, want.value.block)


def test_step_limit():
    cp = L.compile_program(L.compile_source(SPIN))
    with pytest.raises(StepLimitExceeded) as ei:
        L.run(cp, [np.array([0, 5])], depth=8, max_steps=250)
    assert ei.value.limit == 250
    with pytest.raises(StepLimitExceeded):
        L.run(cp, [np.array([0])], depth=8, max_steps=1000)


def test_gather_and_masked_modes_agree(corpus_compiled):
    ins = [np.array([9, 2, 7, 4])]
    a, ta = L.run(corpus_compiled["fibonacci"][2], ins, depth=32, mode="masked")
    b, tb = L.run(corpus_compiled["fibonacci"][2], ins, depth=32, mode="gather")
    assert a.tobytes() == b.tobytes() and ta.steps == tb.steps and ta.stack_ops == tb.stack_ops
    with pytest.raises(ValueError):
        L.run(corpus_compiled["fibonacci"][2], [np.array([1])], depth=8, mode="simd")


def test_debug_mode_and_observer(corpus_compiled):
    for name, (e, _, cp) in corpus_compiled.items():
        if name == "nuts_lite":
            continue
        ins = e.make_inputs(np.random.default_rng(3), 3)
        L.run(cp, ins, depth=64, debug=True)
    seen = []
    _, tr = L.run(corpus_compiled["fibonacci"][2], [np.array([5])], depth=16,
                  observer=lambda m, b, sel: seen.append(b))
    assert len(seen) == tr.step_count


def test_machine_seeding_and_prebuilt_run(corpus_compiled):
    fib = corpus_compiled["fibonacci"][2]
    m = pc_vm.init_machine(fib, [np.array([4, 4])], depth=8)
    assert m.pc.pointers.tolist() == [2, 2]
    assert m.pc.data[0].tolist() == [m.halt_index] * 2
    assert m.pc.data[1].tolist() == [0, 0]
    m = pc_vm.init_machine(fib, [np.array([6])], depth=16)
    assert pc_vm.run_vm(m).tolist() == [13]
    assert not m.active_mask().any()
    out, _ = L.run(fib, [np.array([0, 9])], depth=32)
    assert out.tolist() == [1, 55]


def test_rng_known_answers_on_device():
    g = load_npz("rng_kat.npz")
    assert L.runtime.rng_uniform(g["keys"], g["ctrs"]).tobytes() == g["u"].tobytes()
    assert L.runtime.rng_uniform(g["fkeys"], g["fctrs"]).tobytes() == g["fu"].tobytes()
    u = L.runtime.rng_uniform(np.arange(20000), np.zeros(20000, np.int64))
    assert ((u >= 0) & (u < 1)).all() and abs(u.mean() - 0.5) < 0.01


def test_gaussian_target_kernels_on_device():
    """logpdf in numpy's einsum order is bit-exact; grad within 1e-12 (OpenBLAS order)."""
    e = load_npz("gauss_logpdf.npz")
    for d in (2, 5, 25, 100, 128):
        t = L.correlated_gaussian(d, 0.5)
        x = e[f"x{d}"]
        lp = _native.target_eval(L.device_target(t.name), "logpdf", x)
        assert lp.tobytes() == e[f"lp{d}"].tobytes(), d
        g = _native.target_eval(L.device_target(t.name), "grad", x)
        np.testing.assert_allclose(g, e[f"g{d}"], rtol=1e-12, atol=1e-14)


def test_logreg_target_kernels_on_device():
    g = load_npz("logreg.npz")
    for n, d, seed in ((25, 3, 2), (200, 5, 7), (1000, 25, 0)):
        t = L.logistic_regression(n, d, seed)
        tag = f"lr{n}x{d}s{seed}"
        w = g[f"{tag}_w"]
        dt = L.device_target(t.name)
        np.testing.assert_allclose(_native.target_eval(dt, "logpdf", w), g[f"{tag}_lp"], rtol=1e-12)
        np.testing.assert_allclose(_native.target_eval(dt, "grad", w), g[f"{tag}_g"],
                                   rtol=1e-10, atol=1e-12)


def test_gradients_match_finite_differences():
    """reference test_acceptance.py:273-292, on the device kernels."""
    for t in (L.correlated_gaussian(2, 0.5), L.correlated_gaussian(3, -0.2),
              L.logistic_regression(200, 5, seed=7)):
        dt = L.device_target(t.name)

        def lp(args, _z, dt=dt):
            return _native.target_eval(dt, "logpdf", args[0])

        pts = np.random.default_rng(1).normal(size=(10, t.dim))
        g = _native.target_eval(dt, "grad", pts)
        h = 1e-6
        for i in range(t.dim):
            e = np.zeros(t.dim)
            e[i] = h
            fd = (lp((pts + e,), 10) - lp((pts - e,), 10)) / (2 * h)
            rel = np.abs(g[:, i] - fd) / np.maximum(np.abs(fd), 1e-12)
            assert rel.max() < 1e-5, (t.name, i, rel.max())


def test_leapfrog_per_step_tolerance():
    """Single leaves (L steps) against reference vectors: 1e-12 relative per step."""
    g = load_npz("leapfrog.npz")
    for d, steps in ((2, 1), (2, 4), (100, 1), (100, 4)):
        _, _, cp = nuts_program({"dim": d, "rho": 0.5, "config": dict(leaf_steps=steps, max_depth=6,
                                                                    iterations=1)}, entry="leapfrog")
        tag = f"d{d}_L{steps}"
        got, _ = L.run(cp, [g[f"{tag}_q"], g[f"{tag}_p"], g[f"{tag}_e"]], depth=4)
        want = g[f"{tag}_out"]
        err = np.abs(got - want) / np.maximum(np.abs(want), 1e-300)
        assert (err <= 1e-12 * steps).all() or np.abs(got - want).max() < 1e-13, (tag, err.max())


def test_leapfrog_is_reversible():
    _, _, cp = nuts_program({"dim": 2, "rho": 0.5, "config": dict(max_depth=6, iterations=1)},
                            entry="leapfrog")
    rng = np.random.default_rng(101)
    q0, p0, eps = rng.normal(size=(1, 2)), rng.normal(size=(1, 2)), np.array([0.25])
    fwd, _ = L.run(cp, [q0, p0, eps], depth=4)
    back, _ = L.run(cp, [fwd[:, :2], -fwd[:, 2:], eps], depth=4)
    assert np.abs(back[:, :2] - q0).max() < 1e-10 and np.abs(back[:, 2:] + p0).max() < 1e-10


@pytest.mark.parametrize("case", ["nuts_d2", "nuts_d5", "nuts_d3m", "nuts_d100"])
def test_nuts_golden_traces_exact_and_chains_close(golden_meta, case):
    meta = golden_meta["nuts"][case]
    g = load_npz("nuts_runs.npz")
    cfg, t, cp = nuts_program(meta)
    z, d = meta["z"], meta["dim"]
    ins = [np.zeros((z, d)), g[f"{case}_key"]]
    out, tr, m = L.run(cp, ins, depth=cfg.min_stack_depth, lane_trace_cap=1 << 16,
                       return_machine=True)
    # control: global schedule, per-lane pc sequences and stack traffic are exact
    assert np.array_equal(np.array([[cp.labels.index(s.block), s.active] for s in tr.steps], np.int32),
                          g[f"{case}_steps"])
    want_lanes = split_lanes(g[f"{case}_lane_len"], g[f"{case}_lane_blocks"])
    for lane, seq in enumerate(m.lane_traces()):
        assert np.array_equal(seq, want_lanes[lane]), lane
    assert tr.stack_ops == meta["stack_ops"]
    assert m.useful_grads == meta["useful_grads"] == tr.useful_invocations({t.grad})
    # positions: accumulated over every leapfrog step of the run
    want = g[f"{case}_out"]
    scale = np.maximum(np.abs(want), 1.0)
    assert (np.abs(out - want) / scale).max() < CHAIN_RTOL


@pytest.mark.parametrize("lanes,sched", [(32, "min_pc"), (64, "most_populated"), (128, "min_pc"),
                                         (256, "most_populated")])
def test_multi_group_schedules_do_not_change_lanes(lanes, sched):
    """Lane isolation: any grouping/schedule gives each chain bit-identical results."""
    cfg, t, cp = nuts_program({"dim": 5, "rho": 0.5, "config": dict(max_depth=8, iterations=4)})
    z = 1500
    ins = [np.zeros((z, 5)), np.arange(z, dtype=np.int64) * 104729 + 3]
    base, _ = L.run(cp, [ins[0][:64], ins[1][:64]], depth=cfg.min_stack_depth)
    got, tr = L.run(cp, ins, depth=cfg.min_stack_depth, lanes_per_group=lanes, schedule=sched)
    assert got[:64].tobytes() == base.tobytes()
    ref = oracle_run(cp, [ins[0][64:96], ins[1][64:96]], cfg.min_stack_depth).output
    assert (np.abs(got[64:96] - ref) / np.maximum(np.abs(ref), 1.0)).max() < CHAIN_RTOL
    assert tr.useful_invocations({t.grad}) > 0
    assert 0 < L.utilization(tr, {t.grad}) <= 1


def test_sampler_statistics():
    """reference test_acceptance.py:205-233: 64 lanes x 400 iterations recover the moments."""
    cfg = L.NutsConfig(step_size=0.25, leaf_steps=4, max_depth=6, iterations=400, seed=0)
    t = L.correlated_gaussian(2, 0.5)
    cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
    z = 64
    key = np.random.default_rng(cfg.seed).integers(0, 2**31, size=z).astype(np.int64)
    flat, _ = L.run(cp, [np.zeros((z, 2)), key], depth=cfg.min_stack_depth)
    samples = L.workloads.chain_array(flat, cfg, 2).reshape(-1, 2)
    mean = samples.mean(axis=0)
    cov = np.cov(samples.T)
    assert np.abs(mean).max() < 0.1
    assert np.abs(cov - t.cov).max() < 0.15


# ---- warp engine: interpreter and program-specialised code (codegen) ------------------------


@pytest.mark.parametrize("codegen", [False, "cached"])
def test_warp_engine_corpus_matches_oracle(corpus_compiled, codegen):
    rng = np.random.default_rng(4)
    for name, (e, _, cp) in corpus_compiled.items():
        ins = e.make_inputs(rng, 77)
        ref = oracle_run(cp, ins, 64).output
        got, _ = L.run(cp, ins, depth=64, engine="warp", codegen=codegen)
        assert_matches(got, ref, f"{name} codegen={codegen}")


@pytest.mark.parametrize("codegen", [False, "cached"])
@pytest.mark.parametrize("exact_logpdf", [True, False])
def test_warp_engine_nuts_lanes_exact(codegen, exact_logpdf):
    """Fused leapfrog superblocks + DMMA gradients: every lane's pc trace is the oracle's."""
    from paper_1910_11141_b200 import prebuilt

    for kw in prebuilt.TEST_NUTS:
        kw = dict(kw)
        cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
        z, d = 96, t.dim
        ins = [np.zeros((z, d)), np.arange(z, dtype=np.int64) * 7919 + 11]
        ref = oracle_run(cp, ins, cfg.min_stack_depth, lane_traces=True)
        got, tr, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen=codegen,
                           exact_logpdf=exact_logpdf, lane_trace_cap=1 << 16, return_machine=True)
        for lane, seq in enumerate(m.lane_traces()):
            assert np.array_equal(seq, ref.lane_blocks[lane]), (d, lane)
        assert (np.abs(got - ref.output) / np.maximum(np.abs(ref.output), 1.0)).max() < CHAIN_RTOL
        want = sum(a * 2 * cfg.leaf_steps for b, a in ref.steps if cp.labels[b] == "leapfrog.b2") \
            // (2 * cfg.leaf_steps) * 2
        assert tr.useful_invocations({t.grad}) == m.useful_grads > 0
        assert m.useful_grads == want


def test_pinned_output_pool_never_overwrites_live_results(corpus_compiled):
    """Large outputs come back in page-locked pool buffers (_native.HOST_POOL); a
    buffer is reused only once every array taken from it is gone."""
    _, _, cp = corpus_compiled["fibonacci"]
    z = 1 << 20  # 8 MiB of output: above the pool threshold
    a = np.arange(z, dtype=np.int64) % 11
    b = (np.arange(z, dtype=np.int64) * 7) % 11
    out_a, _ = L.run(cp, [a], depth=64, engine="warp")
    keep = out_a.copy()
    out_b, _ = L.run(cp, [b], depth=64, engine="warp")
    assert np.array_equal(out_a, keep)  # the first result survived the second run
    assert out_a.__array_interface__["data"][0] != out_b.__array_interface__["data"][0]
    ptr_a = out_a.__array_interface__["data"][0]
    del out_a, keep
    out_c, _ = L.run(cp, [a], depth=64, engine="warp")
    assert out_c.__array_interface__["data"][0] == ptr_a  # the released buffer is recycled
    want = oracle_run(cp, [a[:4096]], depth=64).output
    assert np.array_equal(out_c[:4096], want)


def test_fused_leaf_logpdf_matches_recomputed():
    """The superblock's fused leaf logpdf (lowering.fuse_leaf_logpdf, read by the
    codegen build) is bit-identical to warp_gauss recomputing it (interpreter)."""
    from paper_1910_11141_b200 import prebuilt

    for kw in prebuilt.TEST_NUTS:
        kw = dict(kw)
        cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
        z, d = 96, t.dim
        ins = [np.zeros((z, d)), np.arange(z, dtype=np.int64) * 7919 + 11]
        runs = []
        for cg in (False, "cached"):
            got, _, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen=cg,
                              exact_logpdf=False, lane_trace_cap=1 << 16, return_machine=True)
            runs.append((got, [s.copy() for s in m.lane_traces()]))
        assert np.array_equal(runs[0][0], runs[1][0]), d
        assert all(np.array_equal(a, b) for a, b in zip(runs[0][1], runs[1][1])), d


@pytest.mark.parametrize("codegen", [False, "cached"])
def test_warp_engine_logreg_dmma_gradient(codegen):
    """Logistic-regression gradients on the warp engine's fused two-GEMM DMMA path match the
    reference formula (workloads.py:221-228) to 1e-12, and NUTS on that target keeps every
    lane's pc trace equal to the oracle's."""
    from oracle import lockstep_oracle as O
    from paper_1910_11141_b200 import prebuilt

    for n, d, seed in prebuilt.LR_GRAD:
        t, cp = prebuilt.lr_gradient(n, d, seed)
        w = np.random.default_rng(seed).normal(size=(77, d)) * 0.3
        got, _ = L.run(cp, [w], depth=4, engine="warp", codegen=codegen)
        want = O.logreg_grad(w, L.device_target(t.name).params["sx"])
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())
    kw = dict(prebuilt.LR_NUTS)
    cfg, t, cp = prebuilt.lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
    z = 64
    ins = [np.zeros((z, t.dim)), np.arange(z, dtype=np.int64) * 7919 + 11]
    ref = oracle_run(cp, ins, cfg.min_stack_depth, lane_traces=True)
    got, _, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen=codegen,
                      lane_trace_cap=1 << 16, return_machine=True)
    for lane, seq in enumerate(m.lane_traces()):
        assert np.array_equal(seq, ref.lane_blocks[lane]), lane
    assert (np.abs(got - ref.output) / np.maximum(np.abs(ref.output), 1.0)).max() < CHAIN_RTOL


def test_config4_tall_logreg_lanes_exact_on_a_sample():
    """BASELINE config 4 (logistic regression on a 100k x 100 design; sx = 80 MB streams
    through each warp's shared-memory ring by bulk async copies): 40 chains of the bench's
    program through its specialised library — every lane's pc trace equals the oracle's
    (tree depths, U-turns, accepts) and the chains agree within CHAIN_RTOL."""
    from paper_1910_11141_b200 import prebuilt

    kw = dict(prebuilt.CONFIG4)
    cfg, t, cp = prebuilt.lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
    z = 40
    ins = [np.zeros((z, t.dim)), np.arange(z, dtype=np.int64) * 7919 + 11]
    ref = oracle_run(cp, ins, cfg.min_stack_depth, lane_traces=True)
    for exact in (True, False):
        got, _, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen="cached",
                          exact_logpdf=exact, lane_trace_cap=1 << 16, return_machine=True)
        for lane, seq in enumerate(m.lane_traces()):
            assert np.array_equal(seq, ref.lane_blocks[lane]), (exact, lane)
        assert (np.abs(got - ref.output) / np.maximum(np.abs(ref.output), 1.0)).max() < CHAIN_RTOL


def test_warp_engine_logreg_fast_logpdf():
    """Fast mode (exact_logpdf=False): the fused DMMA logistic-regression logpdf agrees with
    the reference formula (workloads.py:216-219) to 1e-12 relative."""
    from oracle import lockstep_oracle as O
    from paper_1910_11141_b200 import prebuilt

    for n, d, seed in prebuilt.LR_GRAD:
        t = L.logistic_regression(n, d, seed)
        cp = L.compile_program(L.compile_source(f"def lp(w) {{ return {t.logpdf}(w); }}", "lp"))
        w = np.random.default_rng(seed + 1).normal(size=(77, d)) * 0.3
        got, _ = L.run(cp, [w], depth=4, engine="warp", exact_logpdf=False)
        want = O.logreg_logpdf(w, L.device_target(t.name).params["sx"])
        np.testing.assert_allclose(got, want, rtol=1e-12)


# ---- BASELINE config 5: ill-conditioned 1000-d gaussian, max_tree_depth 15 ------------------


@pytest.fixture(scope="module")
def illcond_programs():
    """rho = 9999/10999 at d = 1000: covariance eigenvalues 1000/10999 and 10000000/10999,
    condition number 1e4. Step sizes: 0.02 grows deep trees, 0.25 is the
    bench setting, 0.7 puts eps*omega_max above 2 so every trajectory diverges."""
    t = L.correlated_gaussian(1000, 9999 / 10999)
    ev = np.linalg.eigvalsh(t.cov)
    assert abs(ev.max() / ev.min() - 1e4) < 1e-6 * 1e4
    out = {}
    for eps in (0.02, 0.25, 0.7):
        cfg = L.NutsConfig(step_size=eps, leaf_steps=4, max_depth=15, iterations=3, seed=0)
        out[eps] = (cfg, t, L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main")))
    return out


@pytest.mark.parametrize("engine", ["exact", "warp"])
@pytest.mark.parametrize("eps", [0.02, 0.25, 0.7])
def test_illconditioned_1000d_depth15_lanes_exact(illcond_programs, eps, engine):
    cfg, t, cp = illcond_programs[eps]
    z, d = 32, t.dim
    ins = [np.zeros((z, d)), np.arange(z, dtype=np.int64) * 7919 + 11]
    ref = oracle_run(cp, ins, cfg.min_stack_depth, lane_traces=True)
    got, tr, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine=engine, lane_trace_cap=1 << 16,
                       return_machine=True)
    # every tree depth, divergence exit and accept decision is the oracle's
    for lane, seq in enumerate(m.lane_traces()):
        assert np.array_equal(seq, ref.lane_blocks[lane]), (eps, lane)
    # at eps 0.7 only positions that passed the divergence test reach the chain
    assert np.isfinite(got).all()
    assert (np.abs(got - ref.output) / np.maximum(np.abs(ref.output), 1.0)).max() < CHAIN_RTOL
    assert m.useful_grads == tr.useful_invocations({t.grad}) > 0


# ---- round 2: the benchmarked library, the superblock per step, device dot, refill, schedules --


@pytest.mark.parametrize("schedule", ["min_pc", "priority"])
def test_bench_library_lanes_exact_against_reference(golden_meta, schedule):
    """The exact program bench.py times (prebuilt.BENCH: d=100, T=10, depth 10, warp engine,
    specialised library, fast logpdf): every lane's pc trace equals the reference's own
    (observer-recorded, tests/golden nuts_d100_T10) and the chains agree with the reference's
    output; gradient counts are the reference's."""
    from paper_1910_11141_b200 import prebuilt

    meta = golden_meta["nuts"]["nuts_d100_T10"]
    g = load_npz("nuts_runs.npz")
    kw = dict(prebuilt.BENCH)
    assert {k: meta["config"][k] for k in meta["config"]} == {k: kw[k] for k in meta["config"]}
    cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
    z = meta["z"]
    ins = [np.zeros((z, t.dim)), g["nuts_d100_T10_key"]]
    got, tr, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen="cached",
                       exact_logpdf=False, schedule=schedule, lane_trace_cap=1 << 16, return_machine=True)
    assert m._h.program.lib_path.endswith(".so") and "/gen/" in m._h.program.lib_path
    want_lanes = split_lanes(g["nuts_d100_T10_lane_len"], g["nuts_d100_T10_lane_blocks"])
    for lane, seq in enumerate(m.lane_traces()):
        assert np.array_equal(seq, want_lanes[lane]), lane
    want = g["nuts_d100_T10_out"]
    assert (np.abs(got - want) / np.maximum(np.abs(want), 1.0)).max() < CHAIN_RTOL
    assert m.useful_grads == meta["useful_grads"]


@pytest.mark.parametrize("codegen", [False, "cached"])
def test_leapfrog_superblock_per_step_tolerance(codegen):
    """Single leaves through the warp engine's fused DMMA leapfrog superblock (the headline's
    gradient path) against the reference's vectors: 1e-12 relative per leapfrog step, scaled
    by each lane's largest component (reference gradient: OpenBLAS dgemm)."""
    from paper_1910_11141_b200 import prebuilt

    g = load_npz("leapfrog.npz")
    for d, steps in prebuilt.LEAPFROG:
        _, _, cp = prebuilt.nuts(d, 0.5, step_size=0.25, leaf_steps=steps, max_depth=6, iterations=1,
                                 entry="leapfrog")
        tag = f"d{d}_L{steps}"
        got, _, m = L.run(cp, [g[f"{tag}_q"], g[f"{tag}_p"], g[f"{tag}_e"]], depth=4, engine="warp",
                          codegen=codegen, return_machine=True)
        assert any(int(o["opcode"]) == 64 for o in m._dp.ops)  # the fused superblock ran
        want = g[f"{tag}_out"]
        scale = np.abs(want).max(axis=1, keepdims=True)
        err = (np.abs(got - want) / scale).max()
        assert err <= 1e-12 * steps, (tag, err)


@pytest.mark.parametrize("engine", ["exact", "warp"])
def test_device_dot_bit_exact_on_reference_rows(engine):
    """`dot` = numpy's pairwise `(a*b).sum(axis=1)` (reference runtime.py:248-250), bit for
    bit on every row of the reference fixture (n = 1 .. 2500)."""
    g = load_npz("dot_rows.npz")
    cp = L.compile_program(L.compile_source("def f(a, b) { return dot(a, b); }", "f"))
    off = 0
    by_n: dict[int, list] = {}
    for k, n in enumerate(g["lens"].tolist()):
        by_n.setdefault(n, []).append((g["a"][off:off + n], g["b"][off:off + n], g["res"][k]))
        off += n
    for n, rows in by_n.items():
        a = np.stack([r[0] for r in rows])
        b = np.stack([r[1] for r in rows])
        got, _ = L.run(cp, [a, b], depth=4, engine=engine)
        assert got.tobytes() == np.array([r[2] for r in rows]).tobytes(), n


@pytest.mark.parametrize("case", ["nuts_d5", "nuts_d100", "nuts_d3m"])
def test_warp_engine_group_trace_is_the_reference_trace(golden_meta, case):
    """Tracing on the throughput engine: a batch of <= 32 chains is one warp group; with the
    reference's rule and program (min_pc, no fusion, interpreter) its group trace is the
    reference's own ScheduleTrace step for step — block, active lanes — with the same
    per-variable stack-op counts, and it round-trips the reference's JSON wire format."""
    from paper_1910_11141_b200.reference import metrics as RM

    meta = golden_meta["nuts"][case]
    g = load_npz("nuts_runs.npz")
    t = L.correlated_gaussian(meta["dim"], meta["rho"])
    cfg = L.NutsConfig(**meta["config"])
    cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
    ins = [np.zeros((meta["z"], meta["dim"])), g[f"{case}_key"]]
    out, _, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen=False, optimize=False,
                      schedule="min_pc", group_trace_cap=1 << 16, return_machine=True)
    np.testing.assert_allclose(out, g[f"{case}_out"], rtol=CHAIN_RTOL, atol=CHAIN_RTOL)
    trs = m.group_traces()
    assert len(trs) == 1
    want = [tuple(int(v) for v in x) for x in g[f"{case}_steps"]]
    assert [(cp.labels.index(s.block), s.active) for s in trs[0].steps] == want
    assert trs[0].stack_ops == meta["stack_ops"]
    back = RM.trace_from_json(RM.trace_to_json(trs[0]))
    assert back.steps == trs[0].steps and back.stack_ops == trs[0].stack_ops
    assert RM.utilization(trs[0], {t.grad}) == pytest.approx(
        meta["useful_grads"] / (meta["z"] * sum(s.prims.get(t.grad, 0) for s in trs[0].steps)))


def test_group_traces_account_for_every_gradient():
    """The benchmarked library (fused superblocks, paired blocks, priority schedule) on 96
    chains = three groups: the group traces' useful gradient invocations add up to the run's
    useful-gradient count, and each group's utilization is in (0, 1]."""
    from paper_1910_11141_b200 import prebuilt
    from paper_1910_11141_b200.reference import metrics as RM

    kw = dict(prebuilt.BENCH)
    cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
    z = 96
    ins = [np.zeros((z, t.dim)), np.arange(z, dtype=np.int64) * 7919 + 11]
    _, _, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen="cached", exact_logpdf=False,
                    schedule="priority", optimize=True, group_trace_cap=1 << 12, return_machine=True)
    trs = m.group_traces()
    assert len(trs) == 3
    useful = sum(s.active * s.prims.get(t.grad, 0) for tr in trs for s in tr.steps)
    assert useful == m.useful_grads
    for tr in trs:
        assert 0 < RM.utilization(tr, {t.grad}) <= 1


@pytest.mark.parametrize("codegen", [False, "cached"])
def test_warp_engine_nuts_refill(codegen):
    """Chains outnumber the resident lanes 3:1 (4 groups of 32, persistent refill from the
    chain queue): sampled chains from every refill wave equal the oracle's lane for lane."""
    from paper_1910_11141_b200 import prebuilt

    kw = dict(prebuilt.TEST_NUTS[1])  # d=100, T=3
    cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
    z = 3 * 4 * 32
    ins = [np.zeros((z, t.dim)), np.arange(z, dtype=np.int64) * 104729 + 17]
    got, tr, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen=codegen, groups=1,
                       exact_logpdf=False, lane_trace_cap=1 << 14, return_machine=True)
    assert m._h.groups == 4  # 128 resident lanes for 384 chains
    pick = np.r_[0:32, 160:192, 352:384]
    ref = oracle_run(cp, [ins[0][pick], ins[1][pick]], cfg.min_stack_depth, lane_traces=True)
    traces = m.lane_traces()
    for i, lane in enumerate(pick):
        assert np.array_equal(traces[lane], ref.lane_blocks[i]), lane
    assert (np.abs(got[pick] - ref.output) / np.maximum(np.abs(ref.output), 1.0)).max() < CHAIN_RTOL


@pytest.mark.parametrize("name", ["util_z30", "util_z1", "util_d5_z64"])
def test_local_schedule_on_device_reproduces_alg1(golden_meta, name):
    """schedule="local": the device runs paper Alg. 1 (reference local_exec.run_local) on the
    flat program; its gradient utilisation equals the reference local engine's exactly, and
    the pc schedule's equals the reference pc_vm's — the Fig. 6 gate (test_acceptance.py:236-266)."""
    m = golden_meta["local"][name]
    a = load_npz("local_runs.npz")
    t = L.correlated_gaussian(m["dim"], m["rho"])
    cfg = L.NutsConfig(**m["config"])
    cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
    ins = [np.zeros((m["z"], m["dim"])), a[f"{name}_key"]]
    want = a[f"{name}_pc_out"]
    out_l, tr_l = L.run(cp, ins, depth=cfg.min_stack_depth, schedule="local")
    out_p, tr_p = L.run(cp, ins, depth=cfg.min_stack_depth, schedule="min_pc")
    for out in (out_l, out_p):
        assert (np.abs(out - want) / np.maximum(np.abs(want), 1.0)).max() < CHAIN_RTOL
    u_local = L.utilization(tr_l, {t.grad})
    u_pc = L.utilization(tr_p, {t.grad})
    assert u_local == pytest.approx(m["util_local"], rel=1e-12)
    assert u_pc == pytest.approx(m["util_pc"], rel=1e-12)
    if m["z"] == 30:
        assert u_pc / u_local >= 1.5
    if m["z"] == 1:
        assert u_pc == u_local == 1.0


# ---- fp32 arm: tcgen05 (kind::tf32, 3xTF32) leapfrog superblocks, warpgroup stepping -------


@pytest.mark.parametrize("codegen", [False, "cached"])
def test_fp32_leapfrog_per_step_tolerance(codegen):
    """The fp32 arm against the reference's float64 leapfrog vectors: 1e-5 relative per
    leapfrog step (north_star's fp32 contract), scaled by each lane's largest component."""
    from paper_1910_11141_b200 import prebuilt

    g = load_npz("leapfrog.npz")
    for d, steps in prebuilt.LEAPFROG:
        _, _, cp = prebuilt.nuts(d, 0.5, step_size=0.25, leaf_steps=steps, max_depth=6, iterations=1,
                                 entry="leapfrog")
        tag = f"d{d}_L{steps}"
        got, _ = L.run(cp, [g[f"{tag}_q"], g[f"{tag}_p"], g[f"{tag}_e"]], depth=4, engine="warp",
                       codegen=codegen, precision="fp32")
        want = g[f"{tag}_out"]
        err = (np.abs(got - want) / np.abs(want).max(axis=1, keepdims=True)).max()
        assert err <= 1e-5 * steps, (tag, err)
        assert err > 0  # really computed in float32


@pytest.mark.parametrize("codegen", [False, "cached"])
def test_fp32_nuts_control_traces_match_the_f64_oracle(codegen):
    """fp32 arm on NUTS-lite: every lane's block sequence (tree depths, accept and U-turn
    decisions) equals the float64 oracle's, chains agree to float32 accuracy, and the
    warpgroup schedule keeps the reference's gradient count."""
    from paper_1910_11141_b200 import prebuilt

    for kw in prebuilt.TEST_NUTS:
        kw = dict(kw)
        cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
        z, d = 200, t.dim
        ins = [np.zeros((z, d)), np.arange(z, dtype=np.int64) * 7919 + 11]
        ref = oracle_run(cp, ins, cfg.min_stack_depth, lane_traces=True)
        for sched in ("min_pc", "priority", "most_populated"):
            got, tr, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen=codegen,
                               exact_logpdf=False, precision="fp32", schedule=sched,
                               lane_trace_cap=1 << 16, return_machine=True)
            same = sum(np.array_equal(seq, ref.lane_blocks[i]) for i, seq in enumerate(m.lane_traces()))
            assert same == z, (d, sched, same)
            err = (np.abs(got - ref.output) / np.maximum(np.abs(ref.output), 1.0)).max()
            assert err < 1e-4, (d, sched, err)
            want = sum(a * 2 * cfg.leaf_steps for b, a in ref.steps if cp.labels[b] == "leapfrog.b2") \
                // (2 * cfg.leaf_steps) * 2
            assert m.useful_grads == want


def test_fp32_refill_and_faults():
    """fp32 machines refill lanes across warpgroups and report stack overflow like fp64."""
    from paper_1910_11141_b200 import prebuilt

    kw = dict(prebuilt.TEST_NUTS[1])
    cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
    z = 1500
    ins = [np.zeros((z, t.dim)), np.arange(z, dtype=np.int64) * 104729 + 17]
    got, _, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen="cached", groups=1,
                      exact_logpdf=False, precision="fp32", return_machine=True)
    assert m._h.groups % 4 == 0 and m._h.groups * 32 < z
    pick = np.r_[0:16, 700:716, 1484:1500]
    ref = oracle_run(cp, [ins[0][pick], ins[1][pick]], cfg.min_stack_depth)
    assert (np.abs(got[pick] - ref.output) / np.maximum(np.abs(ref.output), 1.0)).max() < 1e-4
    with pytest.raises(StackOverflow):
        L.run(cp, ins, depth=3, engine="warp", codegen="cached", exact_logpdf=False, precision="fp32")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_dispersed_workload_lanes_exact(precision):
    """The bench's random-start workload (prebuilt.DISPERSED: q0 ~ N(0, I), step 0.1) through
    its specialised library: every lane's pc trace equals the float64 oracle's; chains within
    1e-9 (fp64) / 1e-4 (fp32). (The equicorrelated gaussian's U-turn time barely depends on
    the state, so every chain builds trees of the same size here too.)"""
    from paper_1910_11141_b200 import prebuilt
    from paper_1910_11141_b200.distributed import chain_keys

    kw = dict(prebuilt.DISPERSED)
    cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **dict(kw, iterations=kw["iterations"]))
    z = 160
    ins = [np.random.default_rng(1).standard_normal((z, t.dim)), chain_keys(0, z)]
    ref = oracle_run(cp, ins, cfg.min_stack_depth, lane_traces=True)
    got, _, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen="cached", exact_logpdf=False,
                      schedule="priority", precision=precision, lane_trace_cap=1 << 16, return_machine=True)
    for lane, seq in enumerate(m.lane_traces()):
        assert np.array_equal(seq, ref.lane_blocks[lane]), lane
    tol = CHAIN_RTOL if precision == "fp64" else 1e-4
    assert (np.abs(got - ref.output) / np.maximum(np.abs(ref.output), 1.0)).max() < tol
