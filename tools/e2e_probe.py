import time, sys, os
sys.path.insert(0, '.')
import numpy as np
import paper_1910_11141_b200 as L
from paper_1910_11141_b200 import prebuilt
print(open('/sys/kernel/mm/transparent_hugepage/enabled').read().strip())
kw = dict(prebuilt.BENCH); cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
z = 65536
q0 = np.zeros((z, t.dim)); key = np.arange(z, dtype=np.int64) * 7919 + 11
for i in range(3):
    t0 = time.perf_counter()
    out, tr = L.run(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", exact_logpdf=False, codegen=True)
    print("run", time.perf_counter() - t0)
from paper_1910_11141_b200 import pc_vm
m = pc_vm.init_machine(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", optimize=True, exact_logpdf=False, codegen=True)
h = m._h
for i in range(2):
    t0 = time.perf_counter(); h.reset(); t1 = time.perf_counter()
    h.set_input(0, q0.view(np.uint64)); h.set_input(1, key.view(np.uint64)); t2 = time.perf_counter()
    st = h.run(-1); t3 = time.perf_counter()
    o = h.read_output(1000, np.uint64); t4 = time.perf_counter()
    o2 = o.copy(); t5 = time.perf_counter()
    pre = np.empty_like(o); pre.fill(0); t6 = time.perf_counter()
    h.lib.ls_read_output(h.handle, pre.ctypes.data, pre.nbytes); t7 = time.perf_counter()
    print(f"reset {t1-t0:.4f} set_input {t2-t1:.4f} run {t3-t2:.4f} (kernel {st.kernel_ms/1e3:.4f}) read_fresh {t4-t3:.4f} copy {t5-t4:.4f} read_prefaulted {t7-t6:.4f}")
