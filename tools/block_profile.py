"""Cycle-weighted per-block profile of the bench program on the warp engine (dev tool).

Runs one warm launch and prints, per flat block, steps, mean active lanes, total
SM cycles (sum over warps) and share, from the device's clock64 accounting.
usage: python tools/block_profile.py [chains] [codegen 0/1] [schedule] [fp64|fp32]  (builds a LSB_CG_BPROF=1 library)
"""
import os
import sys

import numpy as np

os.environ.setdefault("LSB_CG_BPROF", "1")  # a profiling build of the library (clock64 per block)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import prebuilt  # noqa: E402

z = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
cg = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
sched = sys.argv[3] if len(sys.argv) > 3 else "priority"
prec = sys.argv[4] if len(sys.argv) > 4 else "fp64"
prog = os.environ.get("BP_PROGRAM", "bench")
if prog == "config3":
    kw = dict(prebuilt.CONFIG3)
    cfg, t, cp = prebuilt.lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
elif prog == "config5":
    kw = dict(prebuilt.CONFIG5)
    cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
else:
    kw = dict(prebuilt.BENCH)
    cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
q0 = np.zeros((z, t.dim))
key = np.arange(z, dtype=np.int64) * 7919 + 11
m = L.init_machine(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", optimize=True,
                   exact_logpdf=False, codegen=cg, schedule=sched, precision=prec)
m._h.run(-1)
m._h.reset()
st = m._h.run(-1)
nb = len(cp.flat.blocks)
steps, active = m._h.block_totals(nb)
cyc = m._h.block_cycles(nb)
ops = np.array([int(b["op_count"]) for b in m._dp.blocks])
groups = max(1, (z + 31) // 32)
print(f"{prog}: kernel {st.kernel_ms:.1f} ms, {st.useful_grads / st.kernel_ms / 1e3:.1f} M grads/s, "
      f"grad utilisation {st.useful_grads / max(st.launched_grads, 1):.3f}, "
      f"steps/warp {steps.sum() / groups:.0f}, cycles/warp {cyc.sum() / groups / 1e6:.2f} M")
for b in np.argsort(-cyc)[:20]:
    print(f"{b:3d} {cp.labels[b]:18s} steps/warp {steps[b] / groups:7.1f} lanes/step "
          f"{active[b] / max(steps[b], 1):5.1f} ops {ops[b]:5d} cycles/step {cyc[b] / max(steps[b], 1):9.0f} "
          f"share {100 * cyc[b] / cyc.sum():5.1f}%")
