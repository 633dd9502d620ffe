"""Long runs agree in distribution with the reference (north_star: "moment and ESS checks
against the reference").

Fixtures (tests/golden/make_golden.py `dist_runs`): the reference's own `pc_vm.run` chains
from q0 = 0 for a 5-d correlated gaussian (rho 0.9, 128 chains x 200 iterations) and for
logistic regression 200x5 (64 x 150), plus each target's moment ground truth
(reference workloads.py:126-128 `reference_moments`; the LR one is the reference's own
random-walk estimate, workloads.py:230-249).

Device runs use other chain keys (so nothing is bit-identical) and many more chains. Per
dimension, after a burn-in, the posterior mean and variance must agree with the reference
chains within 5 combined Monte-Carlo standard errors (each side's error from its own ESS,
the estimator of distributed.diagnostics), and the effective sample size per draw — the
sampler's efficiency — must agree within a factor 1.6. The fp32 arm is held to the same
statistical bar (it cannot be bit-exact over 200 iterations).
"""

import numpy as np
import pytest
import torch

from conftest import load_npz
from paper_1910_11141_b200.distributed import chain_keys, diagnostics

BURN = 50
CASES = ["dist_g5", "dist_lr200x5"]


def _stats(samples: np.ndarray):
    """(mean, var, ess per dimension, draws) of chains [c, n, d] after the burn-in."""
    x = samples[:, BURN:, :]
    dg = diagnostics(torch.from_numpy(np.ascontiguousarray(x)))
    return dg.mean, dg.var, dg.ess, x.shape[0] * x.shape[1], dg.rhat


def assert_same_distribution(ref_samples: np.ndarray, got_samples: np.ndarray, tag: str, z: float = 5.0):
    m_r, v_r, e_r, n_r, _ = _stats(ref_samples)
    m_g, v_g, e_g, n_g, rhat = _stats(got_samples)
    assert np.all(rhat < 1.05), (tag, rhat)
    # mean: se^2 = var / ESS;  variance: se^2 ~ 2 var^2 / ESS (gaussian-shaped marginals)
    se_m = np.sqrt(v_r / e_r + v_g / e_g)
    assert np.all(np.abs(m_g - m_r) <= z * se_m), (tag, m_g, m_r, se_m)
    se_v = np.sqrt(2 * v_r ** 2 / e_r + 2 * v_g ** 2 / e_g)
    assert np.all(np.abs(v_g - v_r) <= z * se_v), (tag, v_g, v_r, se_v)
    eff_r, eff_g = e_r / n_r, e_g / n_g
    assert np.all(eff_g / eff_r < 1.6) and np.all(eff_r / eff_g < 1.6), (tag, eff_g, eff_r)


def test_reference_chains_recover_their_ground_truth(golden_meta):
    """Pins the fixture and the comparison: the reference's chains agree with the target's
    moment ground truth within their own Monte-Carlo error (reference test_acceptance.py:205-233
    is the 2-d version of this check)."""
    g = load_npz("dist_runs.npz")
    for name in CASES:
        s = g[f"{name}_samples"]
        meta = golden_meta["dist"][name]
        assert s.shape == (meta["z"], meta["config"]["iterations"], meta["dim"])
        m, v, e, _, _ = _stats(s)
        assert np.all(np.abs(m - g[f"{name}_mean"]) <= 5 * np.sqrt(v / e)), name
        assert np.all(np.abs(v - np.diag(g[f"{name}_cov"])) <= 5 * np.sqrt(2 * v ** 2 / e) + 0.02), name


def test_comparison_rejects_a_biased_sampler():
    """The statistic has power: shifting one coordinate by 0.2 sd, or over-dispersing it,
    fails the check; splitting the same chains in two halves passes."""
    g = load_npz("dist_runs.npz")
    s = g["dist_g5_samples"]
    assert_same_distribution(s[:64], s[64:], "halves")
    shifted = s[64:].copy()
    shifted[..., 2] += 0.2
    with pytest.raises(AssertionError):
        assert_same_distribution(s[:64], shifted, "shifted")
    wide = s[64:].copy()
    wide[..., 1] *= 1.3
    with pytest.raises(AssertionError):
        assert_same_distribution(s[:64], wide, "wide")


def _device_chains(name, golden_meta, z, precision="fp64", codegen=False):
    import paper_1910_11141_b200 as L
    from paper_1910_11141_b200 import workloads

    meta = golden_meta["dist"][name]
    if name.startswith("dist_g5"):
        t = L.correlated_gaussian(5, 0.9)
    else:
        t = L.logistic_regression(200, 5, seed=7)
    cfg = L.NutsConfig(**meta["config"])
    cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
    ins = [np.zeros((z, t.dim)), chain_keys(10_000, 10_000 + z)]
    out, _ = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen=codegen,
                   exact_logpdf=False, precision=precision)
    return workloads.chain_array(out, cfg, t.dim)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_long_run_matches_reference_distribution(golden_meta, name):
    """4096 device chains (warp engine, fast DMMA logpdf) vs the reference's chains."""
    g = load_npz("dist_runs.npz")
    got = _device_chains(name, golden_meta, 4096)
    assert_same_distribution(g[f"{name}_samples"], got, name)


@pytest.mark.gpu
def test_fp32_long_run_matches_reference_distribution(golden_meta):
    """The fp32 arm (tcgen05 3xTF32 superblock) over 200 iterations, same statistical bar."""
    g = load_npz("dist_runs.npz")
    got = _device_chains("dist_g5", golden_meta, 4096, precision="fp32")
    assert_same_distribution(g["dist_g5_samples"], got, "dist_g5 fp32")
