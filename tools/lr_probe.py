"""Tall logistic-regression gradient throughput on the warp engine (dev tool, GPU).

usage: python tools/lr_probe.py [n] [d] [chains ...]
Times the gradient-only program (prebuilt.lr_gradient) and reports the sx bytes each
m-tile pass streams per second (every 8-chain m-tile reads the whole design once).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import prebuilt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 100
zs = [int(x) for x in sys.argv[3:]] or [32, 256, 2048]
t, cp = prebuilt.lr_gradient(n, d, 0)
for z in zs:
    w = np.random.default_rng(0).normal(size=(z, d)) * 0.1
    m = L.init_machine(cp, [w], depth=4, engine="warp", optimize=True, codegen=os.environ.get("LP_CG", "0") != "0")
    m._h.run(-1)
    m._h.reset()
    st = m._h.run(-1)
    passes = sum((min(32, z - 32 * g) + 7) // 8 for g in range((z + 31) // 32))
    gbs = passes * n * d * 8 / (st.kernel_ms / 1e3) / 1e9
    print(f"n={n} d={d} z={z}: {st.kernel_ms:.2f} ms, {passes} m-tile passes, {gbs:.1f} GB/s of sx, "
          f"{z * 4 * n * d / (st.kernel_ms / 1e3) / 1e12:.2f} TFLOP/s", flush=True)
