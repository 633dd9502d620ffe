"""NUTS on Bayesian logistic regression (BASELINE config 3: German-credit shape 1000 x 25,
2^16 chains), warp engine + codegen, fused two-GEMM DMMA gradient (dev tool, GPU).
usage: python tools/lr_bench.py [build]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import codegen, prebuilt  # noqa: E402
from paper_1910_11141_b200.lowering import lower  # noqa: E402
from paper_1910_11141_b200.pc_vm import infer_types  # noqa: E402
from paper_1910_11141_b200.runtime import VType  # noqa: E402

N, D = 1000, 25
cfg, t, cp = prebuilt.lr_nuts(N, D, 0, step_size=0.05, leaf_steps=4, max_depth=10, iterations=5)
if len(sys.argv) > 1 and sys.argv[1] == "build":
    dp = lower(cp, infer_types(cp.flat, [VType("f64", D), VType("i64")]), optimize=True, superblocks=True)
    print(codegen.library_for(dp))
    sys.exit(0)
z = 1 << 16
q0 = np.zeros((z, D))
key = np.arange(z, dtype=np.int64) * 7919 + 11
m = L.init_machine(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", optimize=True,
                   exact_logpdf=False, codegen="cached")
m._h.run(-1)
m._h.reset()
st = m._h.run(-1)
flops = 4 * N * D  # two GEMMs per gradient (margins, then s^T sx)
rate = st.useful_grads / (st.kernel_ms / 1e3)
print(json.dumps({"workload": f"NUTS, logistic regression {N}x{D}, 2^16 chains, 5 iterations, depth 10",
                  "grad_evals_per_s": rate, "ms": st.kernel_ms, "tflops": rate * flops / 1e12,
                  "roofline_frac": rate * flops / 1e12 / 37.0}))
nb = len(cp.flat.blocks)
steps, active = m._h.block_totals(nb)
cyc = m._h.block_cycles(nb)
for b in np.argsort(-cyc)[:8]:
    print(f"{b:3d} {cp.labels[b]:18s} steps/warp {steps[b] / (z // 32):7.1f} cycles/step {cyc[b] / max(steps[b], 1):9.0f} "
          f"share {100 * cyc[b] / cyc.sum():5.1f}%")
