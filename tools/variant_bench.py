"""Time the bench program under codegen option variants (dev tool, GPU).

usage: LSB_CG_<OPT>=v python tools/variant_bench.py [label]   — builds (if needed) and times one
variant of the benchmark library: 2^16 chains, warm-up + 3 timed launches, priority schedule.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import prebuilt  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else "default"
prec = os.environ.get("VB_PRECISION", "fp64")
kw = dict(prebuilt.BENCH)
cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
z = int(os.environ.get("VB_CHAINS", 1 << 16))
q0 = np.zeros((z, t.dim))
key = np.arange(z, dtype=np.int64) * 7919 + 11
m = L.init_machine(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", optimize=True,
                   exact_logpdf=False, codegen=True, schedule="priority", precision=prec)
m._h.run(-1)
ms = []
for _ in range(3):
    m._h.reset()
    st = m._h.run(-1)
    ms.append(st.kernel_ms)
best = min(ms)
print(f"{label:24s} {prec} z={z}: {best:.2f} ms  steps/warp {st.steps}  {st.useful_grads / best / 1e3:.1f} M grads/s  "
      f"frac {st.useful_grads / best * 1e3 * 2e4 / 1e12 / 37.0:.3f}", flush=True)
