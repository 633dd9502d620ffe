"""Target densities on the device; the reference's program generator and corpus.

The NUTS-lite generator (`NutsConfig`, `nuts_lite_source`, `chain_array`),
the target constructors (`correlated_gaussian`, `logistic_regression`), the
`TargetDensity` registry and the corpus are the reference's own
(reference pkg/src/lockstep/workloads.py), used unchanged: the program text,
and hence the compiled flat program and every pc trace, is the reference's.

What the device needs in addition is each target's parameter block, which
the reference keeps only inside its kernel closures: the
precision matrix P and normaliser of a gaussian (`logpdf = norm - 0.5 x'Px`,
`grad = -xP`, workloads.py:174-195) or the label-signed design matrix sx of
a logistic regression (workloads.py:198-253). `device_target` reads them out
of the registered kernels' closure cells (the very arrays the reference
computes with) and caches a `DeviceTarget` that the engine uploads once per
program.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .reference import runtime as _rt
from .reference import workloads as _w

TWO_PI = _w.TWO_PI
FIBONACCI = _w.FIBONACCI
TargetDensity = _w.TargetDensity
registered_targets = _w.registered_targets
correlated_gaussian = _w.correlated_gaussian
logistic_regression = _w.logistic_regression
NutsConfig = _w.NutsConfig
nuts_lite_source = _w.nuts_lite_source
chain_array = _w.chain_array
CorpusProgram = _w.CorpusProgram
corpus = _w.corpus
corpus_program = _w.corpus_program
fibonacci_source = _w.fibonacci_source

TARGET_GAUSSIAN = 1
TARGET_LOGREG = 2


@dataclass
class DeviceTarget:
    """A registered target density as the CUDA VM evaluates it.

    kind TARGET_GAUSSIAN: params {"prec": P (d x d), "norm": float};
    kind TARGET_LOGREG:   params {"sx": sx (n x d)}.
    """

    name: str
    kind: int
    dim: int
    logpdf: str
    grad: str
    params: dict = field(default_factory=dict, repr=False)

    @property
    def grad_flops(self) -> int:
        """Algorithmic FLOPs of one gradient: 2 d^2 (gaussian), 4 n d (logistic)."""
        if self.kind == TARGET_GAUSSIAN:
            return 2 * self.dim * self.dim
        return 4 * self.params["sx"].shape[0] * self.dim


def _closure(fn) -> dict:
    return {n: c.cell_contents for n, c in zip(fn.__code__.co_freevars, fn.__closure__ or ())}


def _kernel_fn(name: str):
    """The user function behind a registered target kernel (`lambda ins, z: f(ins[0])`,
    reference workloads.py:164-167)."""
    outer = _closure(_rt.resolve_kernel(name).fn)
    return next(v for v in outer.values() if callable(v))


_DEVICE: dict[str, DeviceTarget] = {}


def device_target(name: str) -> DeviceTarget | None:
    """The device form of reference target `name` (None when it is not a gaussian or
    logistic-regression density built by the reference constructors)."""
    hit = _DEVICE.get(name)
    if hit is not None:
        return hit
    t = next((t for t in registered_targets() if t.name == name), None)
    if t is None:
        return None
    try:
        grad = _closure(_kernel_fn(t.grad))
        lp = _closure(_kernel_fn(t.logpdf))
    except (KeyError, StopIteration, AttributeError, TypeError):
        return None
    if "prec" in grad and "norm" in lp:
        prec = np.ascontiguousarray(grad["prec"], dtype=np.float64)
        dt = DeviceTarget(t.name, TARGET_GAUSSIAN, t.dim, t.logpdf, t.grad,
                          {"prec": prec, "norm": float(lp["norm"])})
    elif "sx" in grad:
        dt = DeviceTarget(t.name, TARGET_LOGREG, t.dim, t.logpdf, t.grad,
                          {"sx": np.ascontiguousarray(grad["sx"], dtype=np.float64)})
    else:
        return None
    _DEVICE[name] = dt
    return dt


def device_targets() -> dict[str, DeviceTarget]:
    """Every registered target the device can evaluate, by name."""
    out = {}
    for t in registered_targets():
        dt = device_target(t.name)
        if dt is not None:
            out[t.name] = dt
    return out
