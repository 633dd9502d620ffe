"""Break down one end-to-end run() call of the bench workload (dev tool, GPU)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import pc_vm, prebuilt  # noqa: E402

kw = dict(prebuilt.BENCH)
cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
z = 65536
q0 = np.zeros((z, t.dim))
key = np.arange(z, dtype=np.int64) * 7919 + 11
args = dict(depth=cfg.min_stack_depth, engine="warp", exact_logpdf=False, codegen=True)
outs = []
for i in range(4):
    t0 = time.perf_counter()
    out, tr = L.run(cp, [q0, key], **args)
    outs.append(out)
    if len(outs) > 1:
        outs.pop(0)
    print(f"run() {1e3 * (time.perf_counter() - t0):.1f} ms")
# the phases of one call
t0 = time.perf_counter()
m = pc_vm.init_machine(cp, [q0, key], optimize=True, reuse=True, trace=pc_vm.ScheduleTrace(engine="pc", z=z), **args)
t1 = time.perf_counter()
m._h.stream_output_to_host(m._dp.types[m.flat.output].words)
t2 = time.perf_counter()
st = m._h.run(-1)
t3 = time.perf_counter()
o = m.output_value()
t4 = time.perf_counter()
print(f"init_machine+inputs {1e3*(t1-t0):.1f} ms, stream setup {1e3*(t2-t1):.1f}, run {1e3*(t3-t2):.1f} "
      f"(kernel {st.kernel_ms:.1f}), output {1e3*(t4-t3):.1f}")
