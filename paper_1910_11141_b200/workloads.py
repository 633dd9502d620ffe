"""Target densities, the NUTS-lite program generator, and the test corpus.

API mirror of reference `pkg/src/lockstep/workloads.py`:

* `TargetDensity`, `registered_targets`, `correlated_gaussian`,
  `logistic_regression` (`workloads.py:107-253`). A target registers
  `logpdf_<name>` / `grad_<name>` primitives. Unlike the reference, whose
  kernels are numpy closures, these primitives are *device* opcodes: the
  target keeps its parameter block (precision matrix P and normaliser, or the
  label-signed design matrix sx) and the VM evaluates the density on the
  B200. Parameters are built with the same numpy calls as the reference
  (`np.linalg.inv`, `slogdet`, `default_rng(seed)` draws), so they are
  bit-identical on the same numpy build.
* `NutsConfig`, `nuts_lite_source`, `chain_array` (`workloads.py:259-480`):
  the sampler is source text in the package language with every constant
  baked in; it must be character-identical to the reference so the compiled
  flat program (and thus every pc trace) is the same.
* the corpus programs and `corpus()` (`workloads.py:22-97`, `:483-532`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .runtime import F64, OPCODES, DeviceOp, VType, known_kernel, register_kernel

TWO_PI = 6.283185307179586

# ---- corpus programs (plain source text) ------------------------------------------------

FIBONACCI = """\
def fibonacci(n) {
  if (n <= 1) {
    return 1;
  }
  left = fibonacci(n - 1);
  return left + fibonacci(n - 2);
}
"""

COUNTDOWN = """\
def countdown(n) {
  while (0 < n) {
    n = n - 1;
  }
  return n;
}
"""

MUTUAL = """\
def pulse(n) {
  if (n <= 0) {
    return 0;
  }
  return n + echo(n - 1);
}

def echo(n) {
  if (n <= 0) {
    return 1;
  }
  return pulse(n - 1) + 1;
}
"""

TWOSITE = """\
def tally(x) {
  acc = 0;
  while (0 < x) {
    acc = acc + x;
    x = x - 1;
  }
  return acc;
}

def twosite(n) {
  if (n <= 2) {
    a = tally(n + 5);
    return a;
  }
  b = tally(n);
  return b + 1;
}
"""

POLY = """\
def poly(x) {
  a = x * x;
  b = a + x;
  c = b * 2 - x;
  return c + 7;
}
"""

ACKERMANN = """\
def ackermann(m, n) {
  if (m <= 0) {
    return n + 1;
  }
  if (n <= 0) {
    return ackermann(m - 1, 1);
  }
  t = ackermann(m, n - 1);
  return ackermann(m - 1, t);
}
"""


def fibonacci_source() -> str:
    return FIBONACCI


# ---- target densities -----------------------------------------------------------------

TARGET_GAUSSIAN = 1
TARGET_LOGREG = 2


@dataclass
class TargetDensity:
    """A log density exposed to programs as two device primitives.

    `kind` selects the device kernel family; `params` is the parameter block
    the engine uploads once per program: for a gaussian (P, norm) with
    logpdf = norm - 0.5 x'Px and grad = -xP; for logistic regression sx
    (n x d) with logpdf = -sum logaddexp(0, -w sx') - 0.5|w|^2.
    """

    name: str
    dim: int
    logpdf: str
    grad: str
    mean: np.ndarray | None = None
    cov: np.ndarray | None = None
    kind: int = TARGET_GAUSSIAN
    params: dict = field(default_factory=dict, repr=False)
    _moment_fn: Callable[[], tuple[np.ndarray, np.ndarray]] | None = field(default=None, repr=False)

    def reference_moments(self) -> tuple[np.ndarray, np.ndarray]:
        if self.mean is None or self.cov is None:
            self.mean, self.cov = self._moment_fn()
        return self.mean, self.cov

    @property
    def grad_flops(self) -> int:
        """Algorithmic FLOPs of one gradient evaluation."""
        if self.kind == TARGET_GAUSSIAN:
            return 2 * self.dim * self.dim
        n = self.params["sx"].shape[0]
        return 4 * n * self.dim


_TARGETS: dict[str, TargetDensity] = {}


def registered_targets() -> tuple[TargetDensity, ...]:
    return tuple(_TARGETS.values())


def _width_rule(dim: int, scalar_out: bool):
    want = VType("f64", dim)

    def rule(ins):
        (a,) = ins
        if a != want:
            raise TypeError(f"wants an f64 vector of width {dim}, got {a}")
        return F64 if scalar_out else a

    return rule


def _device_fn(target: TargetDensity, which: str):
    def fn(ins, z):
        from . import _native

        return _native.target_eval(target, which, np.ascontiguousarray(ins[0], dtype=np.float64))

    return fn


def _register(t: TargetDensity) -> TargetDensity:
    if t.name in _TARGETS:
        return _TARGETS[t.name]
    if not known_kernel(t.logpdf):
        register_kernel(t.logpdf, 1, _device_fn(t, "logpdf"), _width_rule(t.dim, True),
                        DeviceOp(OPCODES["logpdf"], target=t))
    if not known_kernel(t.grad):
        register_kernel(t.grad, 1, _device_fn(t, "grad"), _width_rule(t.dim, False),
                        DeviceOp(OPCODES["grad"], target=t))
    _TARGETS[t.name] = t
    return t


def correlated_gaussian(dim: int, rho: float) -> TargetDensity:
    """Zero-mean gaussian, unit variances, constant correlation rho."""
    if dim < 1:
        raise ValueError("dim must be at least 1")
    if not -1.0 / max(dim - 1, 1) < rho < 1.0:
        raise ValueError(f"rho={rho} is not a valid equicorrelation for dim={dim}")
    name = f"g{dim}{'p' if rho >= 0 else 'm'}{round(abs(rho) * 1000):03d}"
    if name in _TARGETS:
        return _TARGETS[name]
    cov = np.full((dim, dim), rho, dtype=np.float64)
    np.fill_diagonal(cov, 1.0)
    prec = np.linalg.inv(cov)
    logdet = np.linalg.slogdet(cov)[1]
    norm = -0.5 * (dim * math.log(TWO_PI) + logdet)
    t = TargetDensity(name=name, dim=dim, logpdf=f"logpdf_{name}", grad=f"grad_{name}",
                      mean=np.zeros(dim), cov=cov, kind=TARGET_GAUSSIAN,
                      params={"prec": np.ascontiguousarray(prec), "norm": float(norm)})
    return _register(t)


def _lr_logpdf_host(w: np.ndarray, sx: np.ndarray) -> np.ndarray:
    """Host log density used ONLY by the moment estimator below (test support)."""
    m = w @ sx.T
    return -np.logaddexp(0.0, -m).sum(axis=1) - 0.5 * (w * w).sum(axis=1)


def logistic_regression(n_points: int = 200, n_regressors: int = 5,
                        seed: int = 0) -> TargetDensity:
    """Bayesian logistic posterior on a synthetic design drawn from `seed`."""
    if n_points < 1 or n_regressors < 1:
        raise ValueError("need at least one point and one regressor")
    name = f"lr{n_points}x{n_regressors}s{seed}"
    if name in _TARGETS:
        return _TARGETS[name]
    rng = np.random.default_rng(seed)
    design = rng.normal(size=(n_points, n_regressors))
    w_true = rng.normal(size=n_regressors)
    probs = 1.0 / (1.0 + np.exp(-(design @ w_true)))
    signs = np.where(rng.random(n_points) < probs, 1.0, -1.0)
    sx = np.ascontiguousarray(signs[:, None] * design)

    def moment_fn(walkers: int = 64, sweeps: int = 20_000, burn: int = 4_000):
        # random-walk Metropolis reference moments (reference workloads.py:230-250)
        mrng = np.random.default_rng(seed + 1)
        w = mrng.normal(size=(walkers, n_regressors)) * 0.1
        lp = _lr_logpdf_host(w, sx)
        scale = 0.25 / math.sqrt(n_regressors)
        total = np.zeros(n_regressors)
        outer = np.zeros((n_regressors, n_regressors))
        kept = 0
        for sweep in range(sweeps):
            prop = w + mrng.normal(size=w.shape) * scale
            lp_prop = _lr_logpdf_host(prop, sx)
            accept = np.log(mrng.random(walkers)) < lp_prop - lp
            w = np.where(accept[:, None], prop, w)
            lp = np.where(accept, lp_prop, lp)
            if sweep >= burn:
                total += w.sum(axis=0)
                outer += w.T @ w
                kept += walkers
        mean = total / kept
        return mean, outer / kept - np.outer(mean, mean)

    t = TargetDensity(name=name, dim=n_regressors, logpdf=f"logpdf_{name}", grad=f"grad_{name}",
                      kind=TARGET_LOGREG, params={"sx": sx}, _moment_fn=moment_fn)
    return _register(t)


# ---- NUTS-lite program generation -----------------------------------------------------


@dataclass(frozen=True)
class NutsConfig:
    """Fixed step size, leaf length, doubling cap, kept iterations."""

    step_size: float = 0.25
    leaf_steps: int = 4
    max_depth: int = 6
    iterations: int = 400
    seed: int = 0

    def __post_init__(self):
        if self.leaf_steps < 1:
            raise ValueError("leaf_steps must be at least 1")
        if self.max_depth < 1:
            raise ValueError("max_depth must be at least 1")
        if self.iterations < 1:
            raise ValueError("iterations must be at least 1")
        if not self.step_size > 0:
            raise ValueError("step_size must be positive")

    @property
    def min_stack_depth(self) -> int:
        """Doubling nest + helpers + entry frame (reference workloads.py:280-283)."""
        return self.max_depth + 4


def _vcat_chain(indent: str, stem: str, parts: list[str], returns: bool) -> list[str]:
    """Left-to-right vcat of `parts`, one fresh name per intermediate width."""
    lines, acc = [], parts[0]
    last = len(parts) - 1
    for i in range(1, len(parts)):
        if returns and i == last:
            lines.append(f"{indent}return vcat({acc}, {parts[i]});")
            break
        lines.append(f"{indent}{stem}{i} = vcat({acc}, {parts[i]});")
        acc = f"{stem}{i}"
    return lines


def _normals(k: int) -> list[str]:
    """Box-Muller draws for a k-vector, counters c+0 .. c+2*ceil(k/2)-1."""
    lines, parts = [], []
    pairs = (k + 1) // 2
    for pr in range(pairs):
        a, b = 2 * pr, 2 * pr + 1
        lines.append(f"  u{a} = rng_uniform(key, c + {float(a)!r});")
        lines.append(f"  u{b} = rng_uniform(key, c + {float(b)!r});")
        lines.append(f"  r{pr} = sqrt(0.0 - 2.0 * log(1.0 - u{a}));")
        lines.append(f"  z{a} = r{pr} * cos({TWO_PI!r} * u{b});")
        parts.append(f"vfill:1(z{a})")
        if b < k:
            lines.append(f"  z{b} = r{pr} * sin({TWO_PI!r} * u{b});")
            parts.append(f"vfill:1(z{b})")
    parts.append(f"vfill:1(c + {float(2 * pairs)!r})")
    return lines + _vcat_chain("  ", "pk", parts, True)


_MAIN = """\
def nuts_main(q0, key) {{
  chain = vfill:{width}(0.0);
  c = 0.0;
  q = q0;
  it = 0;
  while (it < {T}) {{
    d = draw_normals(key, c);
    p = vslice:0:{k}(d);
    c = vget(d, {k});
    joint0 = {logpdf}(q) - 0.5 * dot(p, p);
    u0 = rng_uniform(key, c);
    c = c + 1.0;
    logu = joint0 + log(1.0 - u0);
    qm = q;
    pm = p;
    qp = q;
    pp = p;
    prop = q;
    n = 1.0;
    s = 1.0;
    j = 0;
    while (j < {depth} and 0.0 < s) {{
      ud = rng_uniform(key, c);
      c = c + 1.0;
      dir = select(ud < 0.5, 0.0 - 1.0, 1.0);
      if (0.0 < dir) {{
        t = build_tree(qp, pp, dir, j, logu, key, c);
      }} else {{
        t = build_tree(qm, pm, dir, j, logu, key, c);
      }}
      s2 = vget(t, {s_i});
      n2 = vget(t, {n_i});
      c = vget(t, {c_i});
      if (0.0 < dir) {{
        qp = vslice:{k2}:{k3}(t);
        pp = vslice:{k3}:{k4}(t);
      }} else {{
        qm = vslice:0:{k}(t);
        pm = vslice:{k}:{k2}(t);
      }}
      ua = rng_uniform(key, c);
      c = c + 1.0;
      if (0.0 < s2) {{
        accept = ua * n < n2;
        prop = select(accept, vslice:{k4}:{k5}(t), prop);
      }}
      n = n + n2;
      dq = sub(qp, qm);
      sa = select(0.0 <= dot(dq, pm), 1.0, 0.0);
      sb = select(0.0 <= dot(dq, pp), 1.0, 0.0);
      s = s2 * sa * sb;
      j = j + 1;
    }}
    q = prop;
{store}
    it = it + 1;
  }}
  return chain;
}}

def build_tree(q, p, dir, depth, logu, key, c) {{
  if (depth <= 0) {{
    st = leapfrog(q, p, {eps} * dir);
    q1 = vslice:0:{k}(st);
    p1 = vslice:{k}:{k2}(st);
    joint = {logpdf}(q1) - 0.5 * dot(p1, p1);
    n1 = select(logu <= joint, 1.0, 0.0);
    s1 = select(logu < joint + 1000.0, 1.0, 0.0);
{leaf_pack}
  }}
  d2 = depth - 1;
  t1 = build_tree(q, p, dir, d2, logu, key, c);
  s1 = vget(t1, {s_i});
  if (s1 <= 0.0) {{
    return t1;
  }}
  qm = vslice:0:{k}(t1);
  pm = vslice:{k}:{k2}(t1);
  qp = vslice:{k2}:{k3}(t1);
  pp = vslice:{k3}:{k4}(t1);
  prop = vslice:{k4}:{k5}(t1);
  n1 = vget(t1, {n_i});
  c = vget(t1, {c_i});
  if (0.0 < dir) {{
    t2 = build_tree(qp, pp, dir, d2, logu, key, c);
  }} else {{
    t2 = build_tree(qm, pm, dir, d2, logu, key, c);
  }}
  s2 = vget(t2, {s_i});
  n2 = vget(t2, {n_i});
  c = vget(t2, {c_i});
  if (0.0 < dir) {{
    qp = vslice:{k2}:{k3}(t2);
    pp = vslice:{k3}:{k4}(t2);
  }} else {{
    qm = vslice:0:{k}(t2);
    pm = vslice:{k}:{k2}(t2);
  }}
  u = rng_uniform(key, c);
  c = c + 1.0;
  take = u * (n1 + n2) < n2;
  prop = select(take, vslice:{k4}:{k5}(t2), prop);
  dq = sub(qp, qm);
  sa = select(0.0 <= dot(dq, pm), 1.0, 0.0);
  sb = select(0.0 <= dot(dq, pp), 1.0, 0.0);
  s = s2 * sa * sb;
{node_pack}
}}

def draw_normals(key, c) {{
{normals}
}}

def leapfrog(q, p, e) {{
  i = 0;
  while (i < {L}) {{
    g = {grad}(q);
    p = axpy(e / 2.0, g, p);
    q = axpy(e, p, q);
    g = {grad}(q);
    p = axpy(e / 2.0, g, p);
    i = i + 1;
  }}
  return vcat(q, p);
}}
"""


def nuts_lite_source(config: NutsConfig, target: TargetDensity | None = None) -> str:
    """The sampler as source text, constants baked in (reference workloads.py:286-474).

    Inputs per lane: (q0: f64[dim], key: i64); output: f64[iterations*dim].
    Every random draw is rng_uniform(key, c) with c threaded through calls.
    """
    if target is None:
        target = correlated_gaussian(2, 0.5)
    k = target.dim
    store = [f"    base = it * {k};"]
    store += [f"    chain = vstore(chain, base + {i}, vget(q, {i}));" for i in range(k)]
    leaf = _vcat_chain("    ", "lf", ["q1", "p1", "q1", "p1", "q1",
                                      "vfill:1(n1)", "vfill:1(s1)", "vfill:1(c)"], True)
    node = _vcat_chain("  ", "tw", ["qm", "pm", "qp", "pp", "prop",
                                    "vfill:1(n1 + n2)", "vfill:1(s)", "vfill:1(c)"], True)
    return _MAIN.format(
        width=config.iterations * k, T=config.iterations, k=k, k2=2 * k, k3=3 * k,
        k4=4 * k, k5=5 * k, n_i=5 * k, s_i=5 * k + 1, c_i=5 * k + 2,
        depth=config.max_depth, eps=repr(float(config.step_size)), L=config.leaf_steps,
        logpdf=target.logpdf, grad=target.grad, store="\n".join(store),
        leaf_pack="\n".join(leaf), node_pack="\n".join(node), normals="\n".join(_normals(k)))


def chain_array(flat_chain: np.ndarray, config: NutsConfig, dim: int) -> np.ndarray:
    """(lanes, iterations*dim) -> (lanes, iterations, dim)."""
    return flat_chain.reshape(flat_chain.shape[0], config.iterations, dim)


# ---- corpus -------------------------------------------------------------------------------


@dataclass(frozen=True)
class CorpusProgram:
    name: str
    source: str
    entry: str
    make_inputs: Callable[[np.random.Generator, int], list[np.ndarray]]


def _int_inputs(lo: int, hi: int, *, count: int = 1):
    def make(rng, z):
        return [rng.integers(lo, hi, size=z).astype(np.int64) for _ in range(count)]
    return make


TINY_NUTS = NutsConfig(step_size=0.3, leaf_steps=1, max_depth=2, iterations=2)


def _nuts_inputs(dim: int):
    def make(rng, z):
        q0 = rng.normal(size=(z, dim)) * 0.5
        key = rng.integers(0, 2**31, size=z).astype(np.int64)
        return [q0, key]
    return make


def _ackermann_inputs(rng, z):
    return [rng.integers(0, 3, size=z).astype(np.int64),
            rng.integers(0, 4, size=z).astype(np.int64)]


def corpus() -> list[CorpusProgram]:
    """Every program the differential tests run, with input generators."""
    tiny = correlated_gaussian(2, 0.5)
    return [
        CorpusProgram("fibonacci", FIBONACCI, "fibonacci", _int_inputs(0, 11)),
        CorpusProgram("countdown", COUNTDOWN, "countdown", _int_inputs(0, 30)),
        CorpusProgram("mutual", MUTUAL, "pulse", _int_inputs(0, 13)),
        CorpusProgram("twosite", TWOSITE, "twosite", _int_inputs(0, 16)),
        CorpusProgram("poly", POLY, "poly", _int_inputs(-50, 51)),
        CorpusProgram("ackermann", ACKERMANN, "ackermann", _ackermann_inputs),
        CorpusProgram("nuts_lite", nuts_lite_source(TINY_NUTS, tiny), "nuts_main",
                      _nuts_inputs(tiny.dim)),
    ]


def corpus_program(name: str) -> CorpusProgram:
    for p in corpus():
        if p.name == name:
            return p
    raise KeyError(f"no corpus program named '{name}'")
