"""Warp engine vs exact engine on one-op programs at dimension D (dev tool, GPU):
python tools/op_probe.py D CASE"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402

d, case = int(sys.argv[1]), sys.argv[2]
t = L.correlated_gaussian(d, 0.5)
src = {
    "grad": f"def f(q) {{ return {t.grad}(q); }}",
    "logpdf": f"def f(q) {{ return {t.logpdf}(q); }}",
    "dot": "def f(q) { return dot(q, q); }",
    "vcat5": "def f(q) { a = vcat(q, q); b = vcat(a, q); c = vcat(b, a); return c; }",
    "axpy": "def f(q) { return axpy(0.5, q, q); }",
    "leapfrog": f"def f(q) {{ g = {t.grad}(q); p = axpy(0.5, g, q); return vcat(q, p); }}",
}[case]
cp = L.compile_program(L.compile_source(src, "f"))
z = 32
q = np.random.default_rng(0).normal(size=(z, d))
ex, _ = L.run(cp, [q], depth=8, engine="exact")
out, _ = L.run(cp, [q], depth=8, engine="warp")
print("OK", d, case, float(np.abs(out - ex).max()), flush=True)
