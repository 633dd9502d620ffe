"""The CPU oracle is pinned to the reference: bit-exact against golden fixtures.

These run on CPU. They prove the oracle (used as the checker in every GPU
parity test and as the CPU baseline in bench.py) reproduces the reference
engine: corpus outputs, global step traces and stack-op counts, NUTS chains,
per-lane pc traces, rng known answers, dot and einsum summation orders.
"""

import numpy as np
import pytest

import paper_1910_11141_b200 as L
from conftest import load_npz, nuts_program, oracle_run, split_lanes
from oracle import exact_order
from oracle import lockstep_oracle as O


def test_rng_known_answers_survey_a1():
    # SURVEY.md appendix A1 (minted from the reference)
    cases = [(0, 0, 0x0), (1, 1, 0x3FDBDF4BB88FBE54), (7, 3, 0x3FC3DFD6EF8ADA14),
             (123456789, 1048576, 0x3FC2A035AA042FB8), (2147483647, 0, 0x3FE7BA6D240EE410),
             (-5, 17, 0x3FDE420E0559A4C2)]
    for k, c, bits in cases:
        u = O.rng_uniform(np.array([k], np.int64), np.array([c], np.int64))
        assert int(u.view(np.uint64)[0]) == bits


def test_rng_grid_matches_reference():
    g = load_npz("rng_kat.npz")
    assert O.rng_uniform(g["keys"], g["ctrs"]).tobytes() == g["u"].tobytes()
    assert O.rng_uniform(g["fkeys"], g["fctrs"]).tobytes() == g["fu"].tobytes()


def test_exact_order_restatements():
    """The explicit summation orders the CUDA kernels implement."""
    g = load_npz("dot_rows.npz")
    off = 0
    for n, want in zip(g["lens"], g["res"]):
        a, b = g["a"][off:off + n], g["b"][off:off + n]
        off += n
        assert exact_order.dot(a, b) == want, n
    e = load_npz("gauss_logpdf.npz")
    for d in (2, 5, 25, 100, 128):
        t = L.correlated_gaussian(d, 0.5)
        assert np.array_equal(e[f"P{d}"], L.device_target(t.name).params["prec"])
        for row, want in zip(e[f"x{d}"], e[f"lp{d}"]):
            assert exact_order.gauss_logpdf(row, L.device_target(t.name).params["prec"], L.device_target(t.name).params["norm"]) == want, d


def test_corpus_runs_bit_exact(golden_meta, corpus_compiled):
    g = load_npz("corpus_runs.npz")
    for name, meta in golden_meta["corpus"].items():
        _, _, cp = corpus_compiled[name]
        for run in meta["runs"]:
            ins = [g[f"{run['tag']}_in{k}"] for k in range(run["n_inputs"])]
            res = oracle_run(cp, ins, 64)
            assert res.output.tobytes() == g[f"{run['tag']}_out"].tobytes(), run["tag"]
            assert [[cp.labels[b], a] for b, a in res.steps] == run["steps"], run["tag"]
            assert res.stack_ops == run["stack_ops"], run["tag"]


@pytest.mark.parametrize("case", ["nuts_d2", "nuts_d5", "nuts_d3m", "nuts_d100"])
def test_nuts_chains_and_lane_traces_bit_exact(golden_meta, case):
    meta = golden_meta["nuts"][case]
    g = load_npz("nuts_runs.npz")
    cfg, t, cp = nuts_program(meta)
    z, d = meta["z"], meta["dim"]
    key = g[f"{case}_key"]
    res = oracle_run(cp, [np.zeros((z, d)), key], cfg.min_stack_depth, lane_traces=True)
    assert res.output.tobytes() == g[f"{case}_out"].tobytes()
    want_lanes = split_lanes(g[f"{case}_lane_len"], g[f"{case}_lane_blocks"])
    for lane in range(z):
        assert res.lane_blocks[lane] == want_lanes[lane].tolist(), lane
    assert np.array_equal(np.array(res.steps, np.int32), g[f"{case}_steps"])
    assert res.stack_ops == meta["stack_ops"]


def test_leapfrog_vectors_bit_exact():
    g = load_npz("leapfrog.npz")
    for d, steps in ((2, 1), (2, 4), (100, 1), (100, 4)):
        _, _, cp = nuts_program({"dim": d, "rho": 0.5, "config": dict(leaf_steps=steps, max_depth=6,
                                                                    iterations=1)}, entry="leapfrog")
        tag = f"d{d}_L{steps}"
        res = oracle_run(cp, [g[f"{tag}_q"], g[f"{tag}_p"], g[f"{tag}_e"]], 4)
        assert res.output.tobytes() == g[f"{tag}_out"].tobytes(), tag


def test_logreg_target_values():
    g = load_npz("logreg.npz")
    for n, d, seed in ((25, 3, 2), (200, 5, 7), (1000, 25, 0)):
        t = L.logistic_regression(n, d, seed)
        tag = f"lr{n}x{d}s{seed}"
        w = g[f"{tag}_w"]
        assert O.logreg_logpdf(w, L.device_target(t.name).params["sx"]).tobytes() == g[f"{tag}_lp"].tobytes()
        assert O.logreg_grad(w, L.device_target(t.name).params["sx"]).tobytes() == g[f"{tag}_g"].tobytes()


def test_oracle_faults_name_lane_and_block(corpus_compiled):
    cp = corpus_compiled["fibonacci"][2]
    with pytest.raises(O.OracleFault) as ei:
        oracle_run(cp, [np.array([1, 10, 1])], 3)
    assert ei.value.lane == 1 and ei.value.block.startswith("fibonacci.")
