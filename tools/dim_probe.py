"""Warp-engine NUTS at a given dimension with the superblock dimension cap overridden
(dev tool, GPU): python tools/dim_probe.py D [max_superblock_dim]"""
import functools
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import lowering, pc_vm  # noqa: E402

d = int(sys.argv[1])
if len(sys.argv) > 2:
    pc_vm.lower = functools.partial(lowering.lower, max_superblock_dim=int(sys.argv[2]))
cfg = L.NutsConfig(step_size=0.25, leaf_steps=4, max_depth=6, iterations=1, seed=0)
t = L.correlated_gaussian(d, 0.5)
cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
z = 32
ins = [np.zeros((z, d)), np.arange(z, dtype=np.int64) * 7919 + 11]
out, tr = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp")
ex, _ = L.run(cp, ins, depth=cfg.min_stack_depth, engine="exact")
print("OK", sys.argv[1:], tr.step_count, float(np.abs(out - ex).max()), flush=True)
