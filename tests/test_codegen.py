"""Program-specialised block code (codegen.py) on CPU: what gets generated, not run.

* blocks with identical code on different variables (the two direction variants of
  NUTS-lite's tree calls, frame saves and landing pads) are paired into one warp step,
  each lane on its own block's storage; a block's allocs match as a set;
* generation is deterministic and thread-safe (the prebuilt libraries are looked up
  by the hash of the generated text, and build_all generates on several threads).
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from paper_1910_11141_b200 import codegen, prebuilt
from paper_1910_11141_b200.lowering import lower
from paper_1910_11141_b200.pc_vm import infer_types
from paper_1910_11141_b200.runtime import I64, VType


def _bench_dp():
    kw = dict(prebuilt.BENCH)
    cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
    dp = lower(cp, infer_types(cp.flat, [VType("f64", t.dim), I64]), optimize=True, superblocks=True)
    return cp, dp


def test_direction_variants_are_paired():
    cp, dp = _bench_dp()
    pairs = codegen._Gen(dp).find_pairs()
    named = {cp.labels[a]: cp.labels[b] for a, b in pairs.items() if a < b}
    # the tree call sites (qp, pp) / (qm, pm), their landing copies and build_tree's pads
    assert named["nuts_main.b11"] == "nuts_main.b12"
    assert named["nuts_main.b14"] == "nuts_main.b15"
    assert named["build_tree.b10"] == "build_tree.b11"
    # the recursive calls' frame saves: the same stacks allocated, the call on (qp, pp) vs (qm, pm)
    assert named["build_tree.b7"] == "build_tree.b8"
    # empty landing pads pair only with a pad of the same successor
    assert named["nuts_main.r19"] == "nuts_main.r20"
    for a, b in pairs.items():
        if not len(codegen._Gen(dp).block_ops(a)):
            assert int(dp.blocks[a]["a"]) == int(dp.blocks[b]["a"])
    assert all(pairs[b] == a for a, b in pairs.items())  # symmetric, disjoint
    src = codegen.generate(dp)
    assert "const bool sB_ = pc_ == 12;" in src and "case 12: return gb_11(" in src
    assert "__device__ __forceinline__ int gen_pair(int b)" in src
    # the superblock and contraction blocks are never paired
    for b in pairs:
        assert int(dp.blocks[b]["grads"]) == 0


def test_pair_map_rejects_different_code():
    cp, dp = _bench_dp()
    g = codegen._Gen(dp)
    leaf = cp.labels.index("build_tree.b3")
    merge = cp.labels.index("build_tree.b12")
    assert g.pair_map(leaf, merge) is None
    a, b = cp.labels.index("nuts_main.b11"), cp.labels.index("nuts_main.b12")
    pm = g.pair_map(a, b)
    assert pm is not None and len(set(pm.values())) == len(pm)


def test_alloc_sets_map_onto_each_other():
    """b7/b8 save the same eight stacks; the pair's variable map sends A's allocated set
    onto B's and stays a bijection, while the call arguments keep their positional map."""
    cp, dp = _bench_dp()
    g = codegen._Gen(dp)
    a, b = cp.labels.index("build_tree.b7"), cp.labels.index("build_tree.b8")
    pm = g.pair_map(a, b)
    name = dp.var_names
    by = {name[u]: name[v] for u, v in pm.items()}
    assert by["build_tree.qp"] == "build_tree.qm" and by["build_tree.pp"] == "build_tree.pm"
    assert by["build_tree.qm"] == "build_tree.qp" and by["build_tree.pm"] == "build_tree.pp"
    allocs = lambda blk: sorted(int(o["out"]) for o in g.block_ops(blk) if codegen.OP.get(int(o["opcode"])) == "alloc")
    assert sorted(pm[u] for u in allocs(a)) == allocs(b)
    assert len(set(pm.values())) == len(pm)


def test_generation_is_deterministic_across_threads():
    specs = prebuilt.specs()
    dps = [lower(cp, infer_types(cp.flat, ts), optimize=True, superblocks=True) for _, cp, ts in specs]
    serial = [codegen.generate(dp) for dp in dps]
    with ThreadPoolExecutor(8) as ex:
        threaded = list(ex.map(codegen.generate, dps))
    assert serial == threaded
    assert len({hash(s) for s in serial}) == len(set(serial))
    assert np.all([("gb_0(" in s) for s in serial])
