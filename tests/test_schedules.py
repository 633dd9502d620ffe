"""Block-selection rules (paper_1910_11141_b200/schedule.py) on CPU.

* The oracle's restatement of the reference local-static engine (Alg. 1,
  local_exec.run_local) is pinned bit-for-bit to fixtures minted from the
  reference: outputs and the whole batched schedule.
* The flat program run under the `local` rule (what the device executes for
  engine schedule="local") reproduces the local engine's gradient utilisation
  exactly, and the `priority` rule the pc engine's — the Fig. 6 comparison of
  reference test_acceptance.py:236-266.
* Every rule leaves each lane's result bit-identical (lane isolation; reference
  tests/test_local_exec.py:83-88).
"""

import numpy as np
import pytest

import paper_1910_11141_b200 as L
from paper_1910_11141_b200 import ir
from paper_1910_11141_b200 import schedule as S
from conftest import load_npz, oracle_run

CASES = ("util_z30", "util_z1", "util_d5_z64")


def _case(golden_meta, name):
    m = golden_meta["local"][name]
    t = L.correlated_gaussian(m["dim"], m["rho"])
    cfg = L.NutsConfig(**m["config"])
    cg = L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main")
    a = load_npz("local_runs.npz")
    ins = [np.zeros((m["z"], m["dim"])), a[f"{name}_key"]]
    return m, t, cfg, cg, L.compile_program(cg), ins, a


def _grad_counts(cp, t):
    return {b: sum(1 for op in blk.ops if not isinstance(op, ir.Pop) and op.prim.name == t.grad)
            for b, blk in enumerate(cp.flat.blocks)}


def _util(steps, z, counts):
    return sum(a * counts[b] for b, a in steps) / sum(z * counts[b] for b, a in steps)


@pytest.mark.parametrize("name", CASES)
def test_oracle_local_engine_matches_reference(golden_meta, name):
    from oracle import lockstep_oracle as O

    m, t, cfg, cg, cp, ins, a = _case(golden_meta, name)
    out, steps = O.run_local(cg, ins, targets={t.name: L.device_target(t.name)})
    assert out.tobytes() == a[f"{name}_local_out"].tobytes()
    labels = m["local_labels"]
    got = np.array([[labels.index(lbl), act, g] for lbl, act, g in steps], np.int32)
    assert np.array_equal(got, a[f"{name}_local_steps"])
    assert O.utilization(steps, m["z"]) == m["util_local"]


@pytest.mark.parametrize("name", CASES)
def test_local_rule_on_the_flat_program_reproduces_alg1_utilisation(golden_meta, name):
    m, t, cfg, cg, cp, ins, a = _case(golden_meta, name)
    n = len(cp.flat.blocks)
    keys = S.block_keys(cp.flat, cp.labels, "local")
    r = oracle_run(cp, ins, cfg.min_stack_depth, chooser=lambda tops, d: S.select("local", tops, d, keys, n))
    assert r.output.tobytes() == a[f"{name}_pc_out"].tobytes()  # lanes never depend on the rule
    assert _util(r.steps, m["z"], _grad_counts(cp, t)) == m["util_local"]


@pytest.mark.parametrize("name", CASES)
def test_priority_rule_keeps_lanes_and_pc_utilisation(golden_meta, name):
    m, t, cfg, cg, cp, ins, a = _case(golden_meta, name)
    n = len(cp.flat.blocks)
    counts = _grad_counts(cp, t)
    keys = S.block_keys(cp.flat, cp.labels, "priority", [b for b, c in counts.items() if c])
    r = oracle_run(cp, ins, cfg.min_stack_depth, chooser=lambda tops, d: S.select("priority", tops, d, keys, n))
    assert r.output.tobytes() == a[f"{name}_pc_out"].tobytes()
    assert _util(r.steps, m["z"], counts) >= m["util_pc"] - 1e-12
    assert len(r.steps) <= m["pc_step_count"]


def test_fig6_gate_from_the_fixtures(golden_meta):
    """reference test_acceptance.py:256-266: pc/local >= 1.5 at Z=30, both 1.0 at Z=1."""
    g = golden_meta["local"]
    assert g["util_z30"]["util_pc"] / g["util_z30"]["util_local"] >= 1.5
    assert g["util_z1"]["util_pc"] == g["util_z1"]["util_local"] == 1.0


def test_block_keys_shape():
    cfg = L.NutsConfig(step_size=0.25, leaf_steps=4, max_depth=6, iterations=2)
    t = L.correlated_gaussian(2, 0.5)
    cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
    n = len(cp.flat.blocks)
    for rule in ("min_pc", "local", "priority"):
        k = S.block_keys(cp.flat, cp.labels, rule, [39])
        assert k.dtype == np.uint32 and len(k) == n
        assert ((k & 0xFFFF) == np.arange(n)).all()
        assert len(set(k.tolist())) == n
    assert (S.block_keys(cp.flat, cp.labels, "min_pc") == np.arange(n)).all()
    pri = S.block_keys(cp.flat, cp.labels, "priority", [39])
    assert pri[39] >> 16 > pri[cp.flat.entry] >> 16  # contraction blocks run last
    order = S.reverse_post_order(cp.flat, cp.labels)
    assert order[0] == cp.flat.entry and sorted(order) == list(range(n))
    with pytest.raises(ValueError):
        S.block_keys(cp.flat, cp.labels, "fifo")
