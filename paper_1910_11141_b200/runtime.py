"""Lane types and the primitive registry, as seen by the host pipeline.

Mirrors the API of reference `pkg/src/lockstep/runtime.py`:

* `VType`/`F64`/`I64`/`BOOL`, `vtype_of`, `batch` (`runtime.py:32-85`);
* `Kernel`, `register_kernel`, `resolve_kernel`, `known_kernel`,
  `const_name` and the parameterised families `const:`, `vfill:`, `vslice:`
  (`runtime.py:96-119`, `:340-410`);
* the per-primitive static type rules (`runtime.py:122-220`).

What differs is where a kernel *runs*. In the reference each registry entry
carries a numpy batch function. Here every built-in primitive carries a
`DeviceOp` (an opcode of the CUDA VM in `csrc/vm.cuh`) and is only ever
executed inside the B200 engine. Target densities carry a device opcode plus
the target's parameter block (precision matrix / signed design matrix), and
their `fn` evaluates on the GPU through the C ABI. A user kernel registered
with only a numpy `fn` has no device opcode: lowering rejects it loudly
instead of falling back to the CPU.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .errors import StackOverflow, StackUnderflow  # noqa: F401  (re-exported API)

BatchArray = np.ndarray
LaneMask = np.ndarray

_DTYPES = {"f64": np.float64, "i64": np.int64, "bool": np.bool_}


@dataclass(frozen=True)
class VType:
    """Static lane type: dtype kind plus a fixed width (0 means scalar)."""

    kind: str
    width: int = 0

    def __post_init__(self):
        if self.kind not in _DTYPES:
            raise ValueError(f"unknown lane dtype {self.kind!r}")
        if self.width and self.kind != "f64":
            raise ValueError("vector lanes must be f64")

    @property
    def dtype(self):
        return _DTYPES[self.kind]

    @property
    def lane_shape(self) -> tuple[int, ...]:
        return (self.width,) if self.width else ()

    @property
    def words(self) -> int:
        """8-byte words one lane of this type occupies on the device."""
        return self.width if self.width else 1

    def __str__(self):
        return f"f64[{self.width}]" if self.width else self.kind


F64 = VType("f64")
I64 = VType("i64")
BOOL = VType("bool")


def vtype_of(arr: BatchArray) -> VType:
    kinds = {np.dtype(np.float64): "f64", np.dtype(np.int64): "i64", np.dtype(np.bool_): "bool"}
    kind = kinds.get(arr.dtype)
    if kind is None:
        raise TypeError(f"unsupported batch dtype {arr.dtype}")
    return VType(kind, arr.shape[1] if arr.ndim > 1 else 0)


def batch(values, kind: str | None = None) -> BatchArray:
    """Per-lane python values -> a batch array (ints -> i64, reals -> f64)."""
    arr = np.asarray(values)
    if kind is not None:
        return arr.astype(_DTYPES[kind])
    if arr.dtype == np.bool_:
        return arr
    if np.issubdtype(arr.dtype, np.integer):
        return arr.astype(np.int64)
    return arr.astype(np.float64)


def zeros_batch(z: int, vt: VType) -> BatchArray:
    return np.zeros((z,) + vt.lane_shape, dtype=vt.dtype)


# ---- device opcodes ------------------------------------------------------------
# Keep in sync with `enum ls_opcode` in include/lockstep_b200.h.

OPCODES = {
    "const": 1, "id": 2,
    "add": 3, "sub": 4, "mul": 5, "div": 6, "min": 7, "max": 8,
    "le": 9, "lt": 10, "eq": 11,
    "and": 12, "or": 13, "not": 14,
    "neg": 15, "abs": 16,
    "sqrt": 17, "exp": 18, "log": 19, "sin": 20, "cos": 21, "floor": 22,
    "select": 23, "dot": 24, "axpy": 25,
    "vget": 26, "vstore": 27, "vcat": 28, "vfill": 29, "vslice": 30,
    "rng_uniform": 31,
    "logpdf": 32, "grad": 33,
    "leapfrog": 64,  # fused superblock (lowering.match_leapfrog), never a source primitive
    "alloc": 65,     # push of an unobserved save (lowering.dead_saves), never a source primitive
    "normals": 66,   # fused Box-Muller draw function (lowering.match_normals), never a source primitive
}


@dataclass(frozen=True)
class DeviceOp:
    """How the CUDA VM executes a primitive: opcode plus static immediates."""

    opcode: int
    imm0: int = 0
    imm1: int = 0
    fimm: float = 0.0
    target: object | None = None  # TargetDensity for logpdf/grad


@dataclass(frozen=True)
class Kernel:
    """One registered primitive (reference `runtime.py:96-109`).

    `fn(inputs, z)` is the host-callable form. Built-ins have `fn=None`: they
    exist only as VM opcodes. `device` is None for user kernels that only
    registered a numpy function; such programs cannot be lowered.
    """

    name: str
    arity: int
    fn: Callable | None
    type_rule: Callable[[tuple], VType]
    device: DeviceOp | None = None


_REGISTRY: dict[str, Kernel] = {}


def register_kernel(name, arity, fn, type_rule, device: DeviceOp | None = None):
    """Register (or idempotently re-register) a primitive."""
    k = Kernel(name, arity, fn, type_rule, device)
    _REGISTRY[name] = k
    return k


# ---- type rules (reference runtime.py:122-220) --------------------------------


def _same_numeric(ins):
    a, b = ins
    if a != b or a.kind == "bool":
        raise TypeError(f"operands must share a numeric type, got {a} and {b}")
    return a


def _cmp_rule(ins):
    a, b = ins
    if a != b or a.kind == "bool" or a.width:
        raise TypeError(f"comparison needs matching numeric scalars, got {a} and {b}")
    return BOOL


def _eq_rule(ins):
    a, b = ins
    if a != b or a.width:
        raise TypeError(f"eq needs matching scalars, got {a} and {b}")
    return BOOL


def _bool_rule(ins):
    if any(t != BOOL for t in ins):
        raise TypeError("boolean primitive needs bool operands")
    return BOOL


def _float_unary(ins):
    (a,) = ins
    if a.kind != "f64":
        raise TypeError(f"needs f64 lanes, got {a}")
    return a


def _same_unary(ins):
    (a,) = ins
    if a.kind == "bool":
        raise TypeError("needs numeric lanes")
    return a


def _select_rule(ins):
    c, a, b = ins
    if c != BOOL:
        raise TypeError("select condition must be bool")
    if a != b:
        raise TypeError(f"select branches must match, got {a} and {b}")
    return a


def _vec_pair(ins):
    a, b = ins
    if a.kind != "f64" or not a.width or a != b:
        raise TypeError(f"needs two equal f64 vectors, got {a} and {b}")
    return a


def _dot_rule(ins):
    _vec_pair(ins)
    return F64


def _axpy_rule(ins):
    a, x, y = ins
    if a != F64:
        raise TypeError("axpy scale must be f64 scalar")
    return _vec_pair((x, y))


def _vget_rule(ins):
    v, i = ins
    if v.kind != "f64" or not v.width:
        raise TypeError("vget needs an f64 vector")
    if i.width or i.kind == "bool":
        raise TypeError("vget index must be a numeric scalar")
    return F64


def _vstore_rule(ins):
    v, i, x = ins
    _vget_rule((v, i))
    if x != F64:
        raise TypeError("vstore value must be f64 scalar")
    return v


def _vcat_rule(ins):
    a, b = ins
    if a.kind != "f64" or b.kind != "f64" or not a.width or not b.width:
        raise TypeError("vcat needs two f64 vectors")
    return VType("f64", a.width + b.width)


def _rng_rule(ins):
    for t in ins:
        if t.width or t.kind == "bool":
            raise TypeError("rng_uniform needs numeric scalars")
    return F64


def _id_rule(ins):
    return ins[0]


def _builtin(name, arity, rule):
    register_kernel(name, arity, None, rule, DeviceOp(OPCODES[name]))


for _n in ("add", "sub", "mul", "min", "max", "div"):
    _builtin(_n, 2, _same_numeric)
_builtin("le", 2, _cmp_rule)
_builtin("lt", 2, _cmp_rule)
_builtin("eq", 2, _eq_rule)
_builtin("and", 2, _bool_rule)
_builtin("or", 2, _bool_rule)
_builtin("not", 1, _bool_rule)
_builtin("neg", 1, _same_unary)
_builtin("abs", 1, _same_unary)
for _n in ("sqrt", "exp", "log", "sin", "cos", "floor"):
    _builtin(_n, 1, _float_unary)
_builtin("select", 3, _select_rule)
_builtin("dot", 2, _dot_rule)
_builtin("axpy", 3, _axpy_rule)
_builtin("vget", 2, _vget_rule)
_builtin("vstore", 3, _vstore_rule)
_builtin("vcat", 2, _vcat_rule)
_builtin("id", 1, _id_rule)
_builtin("rng_uniform", 2, _rng_rule)


# ---- parameterised families ------------------------------------------------------


def const_name(value) -> str:
    """Canonical const primitive for a python literal (reference `runtime.py:350-357`)."""
    if isinstance(value, bool):
        return "const:bool:" + ("true" if value else "false")
    if isinstance(value, int):
        return f"const:i64:{value}"
    return f"const:f64:{float(value)!r}"


def parse_const(name: str) -> tuple[VType, object]:
    """`const:<kind>:<text>` -> (type, numpy scalar); KeyError when malformed."""
    parts = name.split(":", 2)
    if len(parts) != 3:
        raise KeyError(name)
    _, kind, text = parts
    if kind == "i64":
        return I64, np.int64(int(text))
    if kind == "f64":
        return F64, np.float64(float(text))
    if kind == "bool" and text in ("true", "false"):
        return BOOL, np.bool_(text == "true")
    raise KeyError(name)


def _family(name: str) -> Kernel:
    head = name.split(":", 1)[0]
    if head == "const":
        vt, value = parse_const(name)
        if vt.kind == "f64":
            bits = int(np.float64(value).view(np.int64))
        else:
            bits = int(np.int64(value))
        return Kernel(name, 0, None, lambda ins, _t=vt: _t,
                      DeviceOp(OPCODES["const"], imm0=bits))
    if head == "vfill":
        width = int(name.split(":", 1)[1])
        if width <= 0:
            raise KeyError(name)

        def fill_rule(ins, _w=width):
            if ins[0] != F64:
                raise TypeError("vfill needs an f64 scalar")
            return VType("f64", _w)

        return Kernel(name, 1, None, fill_rule, DeviceOp(OPCODES["vfill"], imm0=width))
    if head == "vslice":
        _, lo_s, hi_s = name.split(":", 2)
        lo, hi = int(lo_s), int(hi_s)
        if not 0 <= lo < hi:
            raise KeyError(name)

        def slice_rule(ins, _lo=lo, _hi=hi):
            (a,) = ins
            if a.kind != "f64" or a.width < _hi:
                raise TypeError(f"vslice:{_lo}:{_hi} needs an f64 vector of width >= {_hi}")
            return VType("f64", _hi - _lo)

        return Kernel(name, 1, None, slice_rule, DeviceOp(OPCODES["vslice"], imm0=lo, imm1=hi))
    raise KeyError(name)


def resolve_kernel(name: str) -> Kernel:
    """Registry lookup that materialises const/vfill/vslice on demand."""
    k = _REGISTRY.get(name)
    if k is None:
        try:
            k = _family(name)
        except ValueError:
            raise KeyError(name) from None
        _REGISTRY[name] = k
    return k


def known_kernel(name: str) -> bool:
    try:
        resolve_kernel(name)
    except (KeyError, ValueError):
        return False
    return True


def rng_uniform(key, counter) -> np.ndarray:
    """Counter-based per-lane uniform on [0, 1), evaluated on the B200.

    Same contract as reference `runtime.py:288-303`: both inputs are hashed
    as int64 (integral f64 counters truncate), so identical (key, counter)
    pairs give identical doubles on every engine.
    """
    from . import _native

    return _native.rng_uniform(np.asarray(key), np.asarray(counter))
