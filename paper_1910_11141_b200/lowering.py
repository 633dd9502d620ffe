"""CompiledProgram -> device program tables for the B200 VM.

The reference engine (`pc_vm.init_machine`, reference `pc_vm.py:140-213`)
turns every flat op into a numpy closure over per-variable storage. Here the
same flat program becomes three plain tables that `include/lockstep_b200.h`
declares (`ls_block`, `ls_op`, `ls_var`) and the CUDA VM interprets, one
thread per lane.

Block indices, terminators and per-block primitive counts are never changed:
pc traces, `ScheduleTrace` records and gradient counts are those of the
reference program. With `optimize=True` (the default when no observer is
attached) two storage passes shrink HBM traffic without changing any lane's
results:

* demote_nonreentrant: variables of functions that cannot be re-entered
  while active (no call cycle through them) need no stack; their
  caller-save pushes and restore pops are identities. `nuts_main.chain`
  (iterations x dim words per slot) is the big win.
* fuse_copies: `update T = f(xs); update V = id T` with T a temporary used
  only there becomes `update V = f(xs)` (in place), e.g. the chain
  `vstore` and every leapfrog `axpy`.

Ops whose output aliases an input in a way that is not elementwise-safe
(`q = grad(q)`) are split through a private scratch temporary.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import ir
from .compiler import CompiledProgram
from .runtime import OPCODES, VType, resolve_kernel

# numpy mirrors of the C structs in include/lockstep_b200.h
OP_DTYPE = np.dtype([("opcode", "<i4"), ("action", "<i4"), ("out", "<i4"), ("nin", "<i4"),
                     ("in", "<i4", (3,)), ("kind", "<i4"), ("width", "<i4"), ("imm0", "<i4"),
                     ("imm1", "<i4"), ("imm2", "<i4"), ("bits", "<i8")])
BLOCK_DTYPE = np.dtype([("op_begin", "<i4"), ("op_count", "<i4"), ("term", "<i4"), ("a", "<i4"),
                        ("b", "<i4"), ("cond", "<i4"), ("grads", "<i4"), ("pad", "<i4")])
VAR_DTYPE = np.dtype([("cls", "<i4"), ("kind", "<i4"), ("width", "<i4"), ("sp", "<i4")])
assert OP_DTYPE.itemsize == 56 and BLOCK_DTYPE.itemsize == 32 and VAR_DTYPE.itemsize == 16

CLASS_CODE = {"stacked": 0, "register": 1, "temporary": 2}
KIND_CODE = {"f64": 0, "i64": 1, "bool": 2}
ACTION_PUSH, ACTION_UPDATE, ACTION_POP = 0, 1, 2
TERM_JUMP, TERM_BRANCH, TERM_PUSHJUMP, TERM_RETURN = 0, 1, 2, 3

# ops whose lane-i output depends only on lane-i inputs (safe to write in place)
_ELEMENTWISE = frozenset({"id", "add", "sub", "mul", "div", "min", "max", "neg", "abs", "sqrt",
                          "exp", "log", "sin", "cos", "floor", "select", "axpy", "le", "lt", "eq",
                          "and", "or", "not", "rng_uniform"})


def _inplace_safe(op, var: str) -> bool:
    name = op.prim.name
    if name in _ELEMENTWISE:
        return True
    if name == "vstore":
        return op.inputs[0] == var and var not in op.inputs[1:]
    if name.startswith("vslice:"):
        return name.split(":")[1] == "0"
    return var not in op.inputs


def grad_names() -> frozenset[str]:
    from .workloads import registered_targets

    return frozenset(t.grad for t in registered_targets())


# ---- storage passes -------------------------------------------------------------------


def recursive_functions(flat: ir.FlatProgram, labels: tuple[str, ...]) -> set[str]:
    """Functions that sit on a call cycle (can be re-entered while active)."""
    fn_of = [lbl.split(".", 1)[0] for lbl in labels]
    calls: dict[str, set[str]] = {}
    for bi, b in enumerate(flat.blocks):
        if isinstance(b.terminator, ir.PushJump):
            calls.setdefault(fn_of[bi], set()).add(fn_of[b.terminator.jump_to])
    out = set()
    for f in set(fn_of):
        seen, todo = set(), list(calls.get(f, ()))
        while todo:
            g = todo.pop()
            if g == f:
                out.add(f)
                break
            if g not in seen:
                seen.add(g)
                todo.extend(calls.get(g, ()))
    return out


def demote_nonreentrant(flat: ir.FlatProgram, classes: dict[str, str], labels) -> tuple:
    """Give stacked variables of non-recursive functions a single register slot."""
    rec = recursive_functions(flat, labels)
    demoted = {v for v, c in classes.items() if c == "stacked" and v.split(".", 1)[0] not in rec}
    if not demoted:
        return flat, classes
    new_classes = {v: ("register" if v in demoted else c) for v, c in classes.items()}
    blocks = []
    for blk in flat.blocks:
        ops = []
        for op in blk.ops:
            if isinstance(op, ir.Pop):
                if op.var not in demoted:
                    ops.append(op)
                continue
            if op.output in demoted:
                if isinstance(op, ir.Push) and op.prim.name == "id" and op.inputs == (op.output,):
                    continue  # caller save of a non-reentrant slot: identity
                ops.append(ir.Update(op.output, op.prim, op.inputs))
                continue
            ops.append(op)
        blocks.append(ir.FlatBlock(tuple(ops), blk.terminator))
    return ir.FlatProgram(tuple(blocks), flat.inputs, flat.output, flat.entry), new_classes


def fuse_copies(flat: ir.FlatProgram, classes: dict[str, str]) -> ir.FlatProgram:
    """`update T = f(xs); update V = id T` (T temporary, single use) -> `update V = f(xs)`."""
    uses: dict[str, int] = {}
    for blk in flat.blocks:
        for op in blk.ops:
            if not isinstance(op, ir.Pop):
                for v in op.inputs:
                    uses[v] = uses.get(v, 0) + 1
        if isinstance(blk.terminator, ir.FlatBranch):
            uses[blk.terminator.cond] = uses.get(blk.terminator.cond, 0) + 1
    blocks = []
    for blk in flat.blocks:
        ops = list(blk.ops)
        out = []
        i = 0
        while i < len(ops):
            op = ops[i]
            nxt = ops[i + 1] if i + 1 < len(ops) else None
            if (isinstance(op, ir.Update) and isinstance(nxt, ir.Update)
                    and classes.get(op.output) == "temporary" and uses.get(op.output, 0) == 1
                    and nxt.prim.name == "id" and nxt.inputs == (op.output,)
                    and op.output != flat.output
                    and (nxt.output not in op.inputs or _inplace_safe(op, nxt.output))):
                out.append(ir.Update(nxt.output, op.prim, op.inputs))
                i += 2
                continue
            out.append(op)
            i += 1
        blocks.append(ir.FlatBlock(tuple(out), blk.terminator))
    return ir.FlatProgram(tuple(blocks), flat.inputs, flat.output, flat.entry)


# ---- table building ------------------------------------------------------------------------


@dataclass
class DeviceProgram:
    """Everything the C ABI needs, plus the host metadata to rebuild traces."""

    compiled: CompiledProgram
    flat: ir.FlatProgram                 # the program the device runs
    classes: dict[str, str]              # its storage classes
    types: dict[str, VType]
    var_names: list[str]
    var_index: dict[str, int]
    blocks: np.ndarray
    ops: np.ndarray
    vars: np.ndarray
    inputs: np.ndarray
    output: int
    targets: list = field(default_factory=list)
    block_prims: list = field(default_factory=list)      # reference per-block prim counts
    block_stack_ops: list = field(default_factory=list)  # reference per-block stack ops
    optimized: bool = False


def _block_prims(flat: ir.FlatProgram) -> list[dict[str, int]]:
    out = []
    for b in flat.blocks:
        counts: dict[str, int] = {}
        for op in b.ops:
            if not isinstance(op, ir.Pop):
                counts[op.prim.name] = counts.get(op.prim.name, 0) + 1
        out.append(counts)
    return out


def _block_stack_ops(flat: ir.FlatProgram, classes: dict[str, str]) -> list[list[tuple[str, str]]]:
    out = []
    for b in flat.blocks:
        rows = []
        for op in b.ops:
            if isinstance(op, ir.Pop):
                rows.append((op.var, "pop"))
            elif classes.get(op.output) == "stacked":
                rows.append((op.output, "push" if isinstance(op, ir.Push) else "update"))
        out.append(rows)
    return out


def lower(compiled: CompiledProgram, types: dict[str, VType], *, optimize: bool = True) -> DeviceProgram:
    """Build the device tables for `compiled` given inferred lane types."""
    flat, classes = compiled.flat, dict(compiled.classes)
    if optimize:
        flat, classes = demote_nonreentrant(flat, classes, compiled.labels)
        flat = fuse_copies(flat, classes)

    grads = grad_names()
    names = sorted(set(classes) | set(types))
    for n in names:
        classes.setdefault(n, "temporary")
    index = {n: i for i, n in enumerate(names)}
    scratch_count = [0]

    def vtype(v: str) -> VType:
        return types.get(v, VType("i64"))

    extra_vars: list[tuple[str, VType]] = []

    def scratch_for(vt: VType) -> int:
        name = f"$scratch{scratch_count[0]}"
        scratch_count[0] += 1
        extra_vars.append((name, vt))
        index[name] = len(names) + len(extra_vars) - 1
        return index[name]

    targets: list = []
    op_rows: list[tuple] = []
    block_rows = []
    ref_prims = _block_prims(compiled.flat)

    for bi, blk in enumerate(flat.blocks):
        begin = len(op_rows)
        for op in blk.ops:
            if isinstance(op, ir.Pop):
                op_rows.append((0, ACTION_POP, index[op.var], 0, [0, 0, 0], 0, 1, 0, 0, 0, 0))
                continue
            k = resolve_kernel(op.prim.name)
            if k.device is None:
                raise NotImplementedError(
                    f"primitive '{op.prim.name}' has no B200 implementation (host-only kernel); "
                    "the lockstep B200 engine has no CPU fallback")
            dev = k.device
            out_vt = vtype(op.output)
            in_kind = KIND_CODE[vtype(op.inputs[0]).kind] if op.inputs else KIND_CODE[out_vt.kind]
            imm0, imm1, bits = dev.imm0, dev.imm1, 0
            if dev.opcode == OPCODES["const"]:
                bits = dev.imm0
                imm0 = 0
            if dev.target is not None:
                if dev.target not in targets:
                    targets.append(dev.target)
                imm0 = targets.index(dev.target)
            action = ACTION_PUSH if isinstance(op, ir.Push) else ACTION_UPDATE
            ins = [index[v] for v in op.inputs]
            row = [dev.opcode, action, index[op.output], len(ins), ins + [0] * (3 - len(ins)),
                   in_kind, out_vt.words, imm0, imm1, 0, bits]
            hazard = (action == ACTION_UPDATE and op.output in op.inputs
                      and not _inplace_safe(op, op.output))
            if hazard:
                tmp = scratch_for(out_vt)
                row[2] = tmp
                op_rows.append(tuple(row))
                op_rows.append((OPCODES["id"], ACTION_UPDATE, index[op.output], 1, [tmp, 0, 0],
                                KIND_CODE[out_vt.kind], out_vt.words, 0, 0, 0, 0))
            else:
                op_rows.append(tuple(row))
        t = blk.terminator
        if isinstance(t, ir.FlatJump):
            term = (TERM_JUMP, t.target, 0, 0)
        elif isinstance(t, ir.FlatBranch):
            term = (TERM_BRANCH, t.true_target, t.false_target, index[t.cond])
        elif isinstance(t, ir.PushJump):
            term = (TERM_PUSHJUMP, t.jump_to, t.return_to, 0)
        else:
            term = (TERM_RETURN, 0, 0, 0)
        g = sum(n for name, n in ref_prims[bi].items() if name in grads)
        block_rows.append((begin, len(op_rows) - begin, term[0], term[1], term[2], term[3], g, 0))

    all_names = names + [n for n, _ in extra_vars]
    all_types = {**{n: vtype(n) for n in names}, **dict(extra_vars)}
    var_arr = np.zeros(len(all_names), dtype=VAR_DTYPE)
    sp_row = 0
    for i, n in enumerate(all_names):
        vt = all_types[n]
        cls = classes.get(n, "temporary")
        var_arr[i] = (CLASS_CODE[cls], KIND_CODE[vt.kind], vt.words, sp_row if cls == "stacked" else -1)
        if cls == "stacked":
            sp_row += 1
    ops = np.zeros(len(op_rows), dtype=OP_DTYPE)
    for i, r in enumerate(op_rows):
        ops[i] = r
    blocks = np.array(block_rows, dtype=BLOCK_DTYPE) if block_rows else np.zeros(0, BLOCK_DTYPE)
    return DeviceProgram(
        compiled=compiled, flat=flat, classes=classes, types=all_types, var_names=all_names,
        var_index={n: i for i, n in enumerate(all_names)}, blocks=blocks, ops=ops, vars=var_arr,
        inputs=np.array([index[v] for v in flat.inputs], dtype=np.int32),
        output=index[flat.output], targets=targets, block_prims=ref_prims,
        block_stack_ops=_block_stack_ops(compiled.flat, compiled.classes), optimized=optimize)
