"""Debug probe: the leapfrog-entry program on each engine vs the reference vectors."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1910_11141_b200 as L
from paper_1910_11141_b200 import prebuilt
g = np.load(os.path.join(ROOT, "tests/golden/leapfrog.npz"))
for d, steps in prebuilt.LEAPFROG:
    _, _, cp = prebuilt.nuts(d, 0.5, step_size=0.25, leaf_steps=steps, max_depth=6, iterations=1, entry="leapfrog")
    tag = f"d{d}_L{steps}"
    ins = [g[f"{tag}_q"], g[f"{tag}_p"], g[f"{tag}_e"]]
    want = g[f"{tag}_out"]
    for eng, cg in (("exact", False), ("warp", False), ("warp", "cached")):
        got, _, m = L.run(cp, ins, depth=4, engine=eng, codegen=cg, return_machine=True)
        err = (np.abs(got - want) / np.abs(want).max(axis=1, keepdims=True)).max()
        print(tag, eng, cg, f"err {err:.3e}", got[0, :4], want[0, :4], flush=True)
