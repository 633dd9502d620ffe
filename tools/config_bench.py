"""Throughput of the BASELINE configs other than the headline one (dev tool, GPU).

  config 3: logistic regression, German-credit shape 1000 x 25, 2^16 chains (prebuilt codegen)
  config 4: logistic regression, 100k x 100 design, one GPU's shard of chains (warp interpreter)
  config 5: ill-conditioned 1000-d gaussian (rho = 9999/10999, condition number 1e4),
            max_tree_depth 15 (warp interpreter)

Each run: warm-up launch, reset, one timed launch (CUDA events around the VM kernel, from
ls_status.kernel_ms); grad evals/s counts useful gradients only.
usage: python tools/config_bench.py [3|4|5 ...] > profiles/r1_configs.jsonl
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import prebuilt  # noqa: E402

FP64_PEAK = 37.0  # TFLOP/s, measured DMMA rate (tools/fp64_peaks.cu)


def timed(cp, cfg, ins, flops, label, **kw):
    t0 = time.time()
    m = L.init_machine(cp, ins, depth=cfg.min_stack_depth, engine="warp", optimize=True,
                       exact_logpdf=False, **kw)
    m._h.run(-1)
    m._h.reset()
    st = m._h.run(-1)
    rate = st.useful_grads / (st.kernel_ms / 1e3)
    nb = len(cp.flat.blocks)
    steps, _ = m._h.block_totals(nb)
    return {"config": label, "chains": int(ins[0].shape[0]), "ms": st.kernel_ms,
            "useful_grads": int(st.useful_grads), "grad_evals_per_s": rate,
            "tflops": rate * flops / 1e12, "roofline_frac": rate * flops / 1e12 / FP64_PEAK,
            "vm_block_steps": int(steps.sum()), "wall_s": time.time() - t0}


def config3():
    n, d = 1000, 25
    cfg, t, cp = prebuilt.lr_nuts(n, d, 0, step_size=0.05, leaf_steps=4, max_depth=10, iterations=5)
    z = 1 << 16
    ins = [np.zeros((z, d)), np.arange(z, dtype=np.int64) * 7919 + 11]
    return timed(cp, cfg, ins, 4 * n * d, "lr 1000x25, eps 0.05, depth 10, 5 iterations, interpreter")


def config4():
    n, d = 100_000, 100
    cfg, t, cp = prebuilt.lr_nuts(n, d, 0, step_size=0.002, leaf_steps=4, max_depth=10, iterations=1)
    z = 1 << 11
    ins = [np.zeros((z, d)), np.arange(z, dtype=np.int64) * 7919 + 11]
    return timed(cp, cfg, ins, 4 * n * d, "lr 100000x100, eps 0.002, depth 10, 1 iteration, interpreter")


def config5():
    cfg, t, cp = prebuilt.nuts(1000, 9999 / 10999, step_size=0.25, leaf_steps=4, max_depth=15,
                               iterations=3)
    z = 1 << 14
    ins = [np.zeros((z, 1000)), np.arange(z, dtype=np.int64) * 7919 + 11]
    return timed(cp, cfg, ins, 2 * 1000 * 1000,
                 "gaussian d=1000 cond 1e4, eps 0.25, depth 15, 3 iterations, interpreter")


if __name__ == "__main__":
    which = sys.argv[1:] or ["3", "4", "5"]
    for w in which:
        try:
            print(json.dumps({"3": config3, "4": config4, "5": config5}[w]()), flush=True)
        except Exception as e:  # noqa: BLE001 - one failing config must not hide the others
            print(json.dumps({"config": w, "error": f"{type(e).__name__}: {e}"}), flush=True)
