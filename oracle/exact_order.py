"""Explicit summation orders of numpy's reductions used on the hot path.

TEST INFRASTRUCTURE ONLY. These restate, as plain Python float arithmetic,
the orders the CUDA kernels implement (csrc/lsb_ops.cuh), so a CPU test can
prove the order itself reproduces numpy bit-for-bit:

* `dot(a, b)` = `(a*b).sum()` (reference runtime.py:248-250): products
  rounded, then `0.0 + pairwise(products)` with numpy's pairwise_sum
  (unroll 8, block 128) — SURVEY.md appendix A2.
* `gauss_logpdf(x, P, norm)` = `norm - 0.5*einsum('zi,ij,zj->z')`
  (reference workloads.py:188-189): terms (x_i*P_ij)*x_j in i-major order,
  summed sequentially in chunks of (8192//d)*d terms — SURVEY.md appendix A3.
"""

from __future__ import annotations


def _pairwise(p: list[float], lo: int, n: int) -> float:
    if n < 8:
        r = 0.0
        for i in range(n):
            r += p[lo + i]
        return r
    if n <= 128:
        r = [p[lo + j] for j in range(8)]
        i = 8
        stop = n - n % 8
        while i < stop:
            for j in range(8):
                r[j] += p[lo + i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += p[lo + i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise(p, lo, n2) + _pairwise(p, lo + n2, n - n2)


def dot(a, b) -> float:
    prods = [float(x) * float(y) for x, y in zip(a, b)]
    return 0.0 + _pairwise(prods, 0, len(prods))


def gauss_logpdf(x, prec, norm: float) -> float:
    d = len(x)
    chunk = (8192 // d) * d if d <= 8192 else d
    xs = [float(v) for v in x]
    acc = s = 0.0
    k = 0
    for i in range(d):
        row = prec[i]
        for j in range(d):
            s += (xs[i] * float(row[j])) * xs[j]
            k += 1
            if k == chunk:
                acc += s
                s = 0.0
                k = 0
    if k:
        acc += s
    return float(norm) - 0.5 * acc
