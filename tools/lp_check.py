import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import paper_1910_11141_b200 as L
from paper_1910_11141_b200 import prebuilt
for kw in prebuilt.TEST_NUTS:
    kw = dict(kw); cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
    z, d = 96, t.dim
    ins = [np.zeros((z, d)), np.arange(z, dtype=np.int64) * 7919 + 11]
    outs = {}
    for cg in (False, "cached"):
        got, tr, m = L.run(cp, ins, depth=cfg.min_stack_depth, engine="warp", codegen=cg, exact_logpdf=False, lane_trace_cap=1 << 16, return_machine=True)
        outs[cg] = (got, [s.copy() for s in m.lane_traces()])
    a, b = outs[False], outs["cached"]
    diff = [i for i in range(z) if not np.array_equal(a[1][i], b[1][i])]
    print(d, 'trace diffs interp vs codegen:', diff[:10], 'max out diff', np.abs(a[0]-b[0]).max())
