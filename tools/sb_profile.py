"""Phase clocks of the fused leapfrog superblock on the bench program (dev tool).

Builds (here) / runs (GPU) the codegen library with LSB_CG_SBPROF=1 and prints,
per superblock call, SM cycles in q staging, p load, kicks, drifts, write-back.
usage: LSB_CG_SBPROF=1 python tools/sb_profile.py [build]
"""
import ctypes as C
import os
import sys

import numpy as np

os.environ["LSB_CG_SBPROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from paper_1910_11141_b200 import codegen, prebuilt  # noqa: E402
from paper_1910_11141_b200.lowering import lower  # noqa: E402
from paper_1910_11141_b200.pc_vm import infer_types  # noqa: E402
from paper_1910_11141_b200.runtime import VType  # noqa: E402

kw = dict(prebuilt.BENCH)
cfg, t, cp = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
if len(sys.argv) > 1 and sys.argv[1] == "build":
    dp = lower(cp, infer_types(cp.flat, [VType("f64", t.dim), VType("i64")]), optimize=True, superblocks=True)
    print(codegen.library_for(dp))
    sys.exit(0)
z = 65536
q0 = np.zeros((z, t.dim))
key = np.arange(z, dtype=np.int64) * 7919 + 11
m = L.init_machine(cp, [q0, key], depth=cfg.min_stack_depth, engine="warp", optimize=True,
                   exact_logpdf=False, codegen="cached")
lib = m._h.lib
lib.ls_debug_sb_profile.argtypes = [C.c_void_p]
buf = (C.c_uint64 * 8)()
m._h.run(-1)
m._h.reset()
lib.ls_debug_sb_profile(buf)
st = m._h.run(-1)
lib.ls_debug_sb_profile(buf)
calls = max(1, buf[5])
print(f"kernel {st.kernel_ms:.1f} ms, superblock calls {calls}")
for i, name in enumerate(["q staging", "p load", "kicks", "drifts", "write-back"]):
    print(f"  {name:12s} {buf[i] / calls:10.0f} cycles/call")
