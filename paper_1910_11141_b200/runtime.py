"""Primitives as the B200 VM executes them.

The reference's runtime (reference pkg/src/lockstep/runtime.py) stays the
type system and kernel registry of the API: `VType`, `vtype_of`, `batch`,
`register_kernel`, `resolve_kernel` and every type rule are the reference's
own, used unchanged. What this module adds is where a primitive *runs*: each
built-in primitive, parameterised family (`const:`, `vfill:`, `vslice:`) and
target kernel (`logpdf_<t>`, `grad_<t>`) maps to a `DeviceOp`, an opcode of
the CUDA VM (`enum ls_opcode` in include/lockstep_b200.h). A kernel the user
registered with only a numpy function has no device opcode: lowering rejects
it loudly instead of falling back to the CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .reference import runtime as _rt

VType = _rt.VType
F64, I64, BOOL = _rt.F64, _rt.I64, _rt.BOOL
vtype_of = _rt.vtype_of
batch = _rt.batch
register_kernel = _rt.register_kernel
resolve_kernel = _rt.resolve_kernel
known_kernel = _rt.known_kernel


def words(vt: VType) -> int:
    """8-byte words one lane of this type occupies on the device."""
    return vt.width if vt.width else 1


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

_BUILTIN = frozenset({"id", "add", "sub", "mul", "div", "min", "max", "le", "lt", "eq", "and", "or",
                      "not", "neg", "abs", "sqrt", "exp", "log", "sin", "cos", "floor", "select",
                      "dot", "axpy", "vget", "vstore", "vcat", "rng_uniform"})


@dataclass(frozen=True)
class DeviceOp:
    """How the CUDA VM executes a primitive: opcode plus static immediates."""

    opcode: int
    imm0: int = 0
    imm1: int = 0
    target: object | None = None  # workloads.DeviceTarget for logpdf/grad


def _const_bits(name: str) -> int:
    _, kind, text = name.split(":", 2)
    if kind == "f64":
        return int(np.float64(float(text)).view(np.int64))
    if kind == "i64":
        return int(np.int64(int(text)))
    if kind == "bool" and text in ("true", "false"):
        return int(text == "true")
    raise KeyError(name)


def device_op(name: str) -> DeviceOp | None:
    """The VM opcode of primitive `name`, or None when it has no device implementation
    (the reference registry still knows it, so type inference works)."""
    if name in _BUILTIN:
        return DeviceOp(OPCODES[name])
    head = name.split(":", 1)[0]
    if head == "const":
        return DeviceOp(OPCODES["const"], imm0=_const_bits(name))
    if head == "vfill":
        return DeviceOp(OPCODES["vfill"], imm0=int(name.split(":")[1]))
    if head == "vslice":
        _, lo, hi = name.split(":")
        return DeviceOp(OPCODES["vslice"], imm0=int(lo), imm1=int(hi))
    for prefix, op in (("logpdf_", "logpdf"), ("grad_", "grad")):
        if name.startswith(prefix):
            from .workloads import device_target

            t = device_target(name[len(prefix):])
            return None if t is None else DeviceOp(OPCODES[op], target=t)
    return None


def rng_uniform(key, counter) -> np.ndarray:
    """Counter-based per-lane uniform on [0, 1), evaluated on the B200.

    Same contract as reference `runtime.py:288-303`: both inputs are hashed
    as int64 (integral f64 counters truncate), so identical (key, counter)
    pairs give identical doubles on every engine.
    """
    from . import _native

    return _native.rng_uniform(np.asarray(key), np.asarray(counter))
