"""Gradient evals/s vs number of chains (BASELINE config 2: 2^10 .. 2^20 chains, fp64, 1 B200).

Same workload as bench.py (NUTS-lite, 100-d correlated gaussian, 10 iterations, depth 10);
device time of the VM launch (CUDA events), inputs resident. Writes one JSON line per chain
count and a summary to profiles/ when --out is given.
usage: python tools/chain_sweep.py [--out profiles/r1_chain_sweep.json] [--max-log2 20]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import prebuilt  # noqa: E402

PEAK = 37.0  # TFLOP/s, measured fp64 DMMA peak (tools/fp64_peaks.cu)

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--min-log2", type=int, default=10)
ap.add_argument("--max-log2", type=int, default=20)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
kw = dict(prebuilt.BENCH)
cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
rows = []
for lg in range(args.min_log2, args.max_log2 + 1):
    z = 1 << lg
    q0 = np.zeros((z, t.dim))
    key = np.arange(z, dtype=np.int64) * 7919 + 11
    m = L.init_machine(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", optimize=True,
                       exact_logpdf=False, codegen=True)
    m._h.run(-1)  # warm-up
    ms, grads = [], 0
    for _ in range(args.reps):
        m._h.reset()
        st = m._h.run(-1)
        ms.append(st.kernel_ms)
        grads += st.useful_grads
    sec = sum(ms) / 1e3
    rate = grads / sec
    row = {"chains": z, "grad_evals_per_s": rate, "ms_per_launch": float(np.mean(ms)),
           "tflops": rate * L.device_target(t.name).grad_flops / 1e12, "roofline_frac": rate * L.device_target(t.name).grad_flops / 1e12 / PEAK}
    rows.append(row)
    print(json.dumps(row), flush=True)
    del m
if args.out:
    json.dump({"workload": "NUTS-lite, 100-d correlated gaussian (rho 0.5), 10 iterations, depth 10, fp64",
               "engine": "warp + codegen", "peak_tflops": PEAK, "sweep": rows}, open(args.out, "w"), indent=1)
