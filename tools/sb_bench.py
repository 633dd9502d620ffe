"""The fused leapfrog superblock alone: 30 leapfrog calls per chain (dev tool).

usage: python tools/sb_bench.py build   (here; with LSB_CG_SBPROF=1 for phase clocks)
       python tools/sb_bench.py          (GPU)
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import codegen, workloads as W  # noqa: E402
from paper_1910_11141_b200.lowering import lower  # noqa: E402
from paper_1910_11141_b200.pc_vm import infer_types  # noqa: E402
from paper_1910_11141_b200.runtime import VType  # noqa: E402

t = W.correlated_gaussian(100, 0.5)
src = f"""
def main(q0, key) {{
  q = q0; p = q0; i = 0;
  while (i < 30) {{
    st = leapfrog(q, p, 0.01);
    q = vslice:0:100(st);
    p = vslice:100:200(st);
    i = i + 1;
  }}
  return q;
}}
def leapfrog(q, p, e) {{
  i = 0;
  while (i < 4) {{
    g = {t.grad}(q);
    p = axpy(e / 2.0, g, p);
    q = axpy(e, p, q);
    g = {t.grad}(q);
    p = axpy(e / 2.0, g, p);
    i = i + 1;
  }}
  return vcat(q, p);
}}
"""
cp = L.compile_program(L.compile_source(src, "main"))
if len(sys.argv) > 1 and sys.argv[1] == "build":
    dp = lower(cp, infer_types(cp.flat, [VType("f64", 100), VType("i64")]), optimize=True, superblocks=True)
    print(codegen.library_for(dp))
    sys.exit(0)
z = 65536
rng = np.random.default_rng(0)
q0 = rng.normal(size=(z, 100))
key = np.arange(z, dtype=np.int64)
m = L.init_machine(cp, [q0, key], depth=4, engine="warp", optimize=True, exact_logpdf=False, codegen="cached")
m._h.run(-1)
m._h.reset()
prof = os.environ.get("LSB_CG_SBPROF") == "1"
buf = (C.c_uint64 * 8)()
if prof:
    m._h.lib.ls_debug_sb_profile.argtypes = [C.c_void_p]
    m._h.lib.ls_debug_sb_profile(buf)
st = m._h.run(-1)
calls = z // 32 * 30
print(f"kernel {st.kernel_ms:.2f} ms, {st.useful_grads / st.kernel_ms / 1e3:.1f} M grads/s, "
      f"{st.useful_grads * 2e4 / st.kernel_ms / 1e9:.2f} TFLOP/s")
if prof:
    m._h.lib.ls_debug_sb_profile(buf)
    n = max(1, buf[5])
    for i, name in enumerate(["q staging", "p load", "kicks", "drifts", "write-back"]):
        print(f"  {name:12s} {buf[i] / n:10.0f} cycles/call")
