"""codegen vs interpreter vs oracle on the warp engine (dev tool)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1910_11141_b200 as L
from conftest import oracle_run

for e in L.corpus():
    cp = L.compile_program(L.compile_source(e.source, e.entry))
    ins = e.make_inputs(np.random.default_rng(4), 77)
    ref = oracle_run(cp, ins, 64).output
    got, _ = L.run(cp, ins, depth=64, engine="warp", codegen=True)
    ok = np.array_equal(got, ref) if got.dtype.kind != "f" else np.allclose(got, ref, rtol=1e-12, atol=0)
    print(e.name, "codegen ok" if ok else "MISMATCH", flush=True)
for d, T, z in ((2, 10, 100), (100, 3, 100)):
    cfg = L.NutsConfig(step_size=0.25, leaf_steps=4, max_depth=10, iterations=T)
    t = L.correlated_gaussian(d, 0.5)
    cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
    q0 = np.zeros((z, d)); key = np.arange(z, dtype=np.int64) * 7919 + 11
    ref = oracle_run(cp, [q0, key], cfg.min_stack_depth, lane_traces=True)
    got, tr, m = L.run(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", codegen=True,
                       exact_logpdf=False, lane_trace_cap=100000, return_machine=True)
    err = np.max(np.abs(got - ref.output) / np.maximum(np.abs(ref.output), 1.0))
    lt = m.lane_traces()
    same = sum(np.array_equal(lt[i], ref.lane_blocks[i]) for i in range(z))
    print(f"nuts d={d}: err {err:.2e} lanes {same}/{z} grads {tr.useful_invocations({t.grad})}", flush=True)
cfg = L.NutsConfig(step_size=0.25, leaf_steps=4, max_depth=10, iterations=10)
t = L.correlated_gaussian(100, 0.5)
cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
z = 65536
q0 = np.zeros((z, 100)); key = np.arange(z, dtype=np.int64) * 7919 + 11
for cg in (False, True):
    m = L.init_machine(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", optimize=True,
                       exact_logpdf=False, codegen=cg)
    m._h.run(-1); m._h.reset(); st = m._h.run(-1)
    print(f"z={z} codegen={cg}: {st.kernel_ms:.1f} ms {st.useful_grads / st.kernel_ms / 1e3:.1f} M grads/s "
          f"{st.useful_grads * 2e4 / st.kernel_ms / 1e9:.2f} TFLOP/s", flush=True)
