"""Warp-engine probe: parity vs oracle + timing (dev tool)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1910_11141_b200 as L
from conftest import oracle_run

for d, T in ((2, 10), (5, 5), (100, 3)):
    cfg = L.NutsConfig(step_size=0.25, leaf_steps=4, max_depth=10, iterations=T)
    t = L.correlated_gaussian(d, 0.5)
    cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
    z = 100
    q0 = np.zeros((z, d)); key = np.arange(z, dtype=np.int64) * 7919 + 11
    ref = oracle_run(cp, [q0, key], cfg.min_stack_depth, lane_traces=True)
    for opt in (False, True):
        for sched in ("min_pc", "most_populated"):
            for exact in (True, False):
                got, tr, m = L.run(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", optimize=opt,
                                   schedule=sched, lane_trace_cap=100000, exact_logpdf=exact, return_machine=True)
                err = np.max(np.abs(got - ref.output) / np.maximum(np.abs(ref.output), 1.0))
                lt = m.lane_traces()
                same = sum(np.array_equal(lt[i], ref.lane_blocks[i]) for i in range(z))
                print(f"d={d} opt={opt} sched={sched} exact_lp={exact}: err={err:.2e} lanes_equal={same}/{z} "
                      f"grads={m.useful_grads}", flush=True)
# timing at scale
for d, T, z in ((100, 10, 65536), (100, 10, 16384)):
    cfg = L.NutsConfig(step_size=0.25, leaf_steps=4, max_depth=10, iterations=T)
    t = L.correlated_gaussian(d, 0.5)
    cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
    q0 = np.zeros((z, d)); key = np.arange(z, dtype=np.int64) * 7919 + 11
    for exact in (True, False):
        for sched in ("min_pc", "most_populated"):
            m = L.init_machine(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", optimize=True,
                               schedule=sched, exact_logpdf=exact)
            st = m._h.run(-1)
            m._h.reset(); st = m._h.run(-1)
            print(f"z={z} exact_lp={exact} sched={sched}: {st.kernel_ms:.1f} ms, grads {st.useful_grads}, "
                  f"{st.useful_grads / st.kernel_ms * 1e3 / 1e6:.1f} M grads/s, "
                  f"{st.useful_grads * 2 * d * d / st.kernel_ms / 1e9:.2f} TFLOP/s", flush=True)
