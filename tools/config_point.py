"""One BASELINE config point on the warp engine + prebuilt library (dev tool, GPU).

usage: python tools/config_point.py config3|config4|config5|dispersed [chains] [fp64|fp32]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import prebuilt  # noqa: E402
from paper_1910_11141_b200.distributed import chain_keys  # noqa: E402

which = sys.argv[1]
z = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 14
prec = sys.argv[3] if len(sys.argv) > 3 else "fp64"
if which == "config3":
    kw = dict(prebuilt.CONFIG3)
    cfg, t, cp = prebuilt.lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
    q0 = np.zeros((z, t.dim))
elif which == "config4":
    kw = dict(prebuilt.CONFIG4)
    cfg, t, cp = prebuilt.lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
    q0 = np.zeros((z, t.dim))
elif which == "config5":
    kw = dict(prebuilt.CONFIG5)
    cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
    q0 = np.zeros((z, t.dim))
else:
    kw = dict(prebuilt.DISPERSED)
    cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
    q0 = np.random.default_rng(1).standard_normal((z, t.dim))
m = L.init_machine(cp, [q0, chain_keys(0, z)], depth=cfg.min_stack_depth, engine="warp", optimize=True,
                   exact_logpdf=False, codegen="cached", schedule="priority", precision=prec)
m._h.run(-1)
m._h.reset()
st = m._h.run(-1)
dt = L.device_target(t.name)
v = st.useful_grads / (st.kernel_ms / 1e3)
print(f"{which} z={z} {prec}: {st.kernel_ms:.1f} ms, {st.useful_grads} grads, {v / 1e6:.2f} M grads/s, "
      f"{v * dt.grad_flops / 1e12:.2f} TFLOP/s = {v * dt.grad_flops / 1e12 / 37.0:.3f} of fp64 peak", flush=True)
