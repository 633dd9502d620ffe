"""One warp-engine launch of the bench workload (for ncu)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L
z = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = L.NutsConfig(step_size=0.25, leaf_steps=4, max_depth=10, iterations=T)
t = L.correlated_gaussian(100, 0.5)
cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
q0 = np.zeros((z, 100)); key = np.arange(z, dtype=np.int64) * 7919 + 11
m = L.init_machine(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", optimize=True, exact_logpdf=False)
st = m._h.run(-1)
m._h.reset()
st = m._h.run(-1)
print(f"{st.kernel_ms:.1f} ms grads {st.useful_grads}", flush=True)
tot_s, tot_a = m._h.block_totals(41)
for b in np.argsort(-tot_s)[:12]:
    print(b, cp.labels[b], int(tot_s[b]), int(tot_a[b]), f"{tot_a[b] / max(tot_s[b], 1):.1f} lanes/step")
ops_per_block = np.array([int(b["op_count"]) for b in m._dp.blocks])
tot_ops = (tot_s * ops_per_block).sum()
groups = max(1, (z + 31) // 32)
print(f"ops executed per warp: {tot_ops / groups:.0f}; steps per warp {tot_s.sum() / groups:.0f}")
print("top blocks by ops:", [(cp.labels[b], int(tot_s[b] * ops_per_block[b] / groups)) for b in np.argsort(-(tot_s * ops_per_block))[:8]])
