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
from .runtime import OPCODES, VType, device_op, words

# numpy mirrors of the C structs in include/lockstep_b200.h
OP_DTYPE = np.dtype([("opcode", "<i4"), ("action", "<i4"), ("out", "<i4"), ("nin", "<i4"),
                     ("in", "<i4", (3,)), ("kind", "<i4"), ("width", "<i4"), ("imm0", "<i4"),
                     ("imm1", "<i4"), ("imm2", "<i4"), ("bits", "<i8")])
BLOCK_DTYPE = np.dtype([("op_begin", "<i4"), ("op_count", "<i4"), ("term", "<i4"), ("a", "<i4"),
                        ("b", "<i4"), ("cond", "<i4"), ("grads", "<i4"), ("pad", "<i4")])
VAR_DTYPE = np.dtype([("cls", "<i4"), ("kind", "<i4"), ("width", "<i4"), ("sp", "<i4"),
                      ("row", "<i4"), ("pad", "<i4")])
assert OP_DTYPE.itemsize == 56 and BLOCK_DTYPE.itemsize == 32 and VAR_DTYPE.itemsize == 24

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


def _registered():
    from .workloads import registered_targets

    return registered_targets()


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


def demote_unpushed(flat: ir.FlatProgram, classes: dict[str, str]) -> tuple:
    """A stacked variable that is never pushed nor popped keeps pointer 1 forever:
    its top is always slot 0, i.e. it is a register (e.g. `build_tree._ret`)."""
    touched = set()
    for blk in flat.blocks:
        for op in blk.ops:
            if isinstance(op, ir.Pop):
                touched.add(op.var)
            elif isinstance(op, ir.Push):
                touched.add(op.output)
    demoted = {v for v, c in classes.items() if c == "stacked" and v not in touched}
    if not demoted:
        return flat, classes
    return flat, {v: ("register" if v in demoted else c) for v, c in classes.items()}


def dead_saves(flat: ir.FlatProgram, classes: dict[str, str], labels) -> set[tuple[int, int]]:
    """Caller saves `push v = id v` whose copied value is never observed.

    A save gives the callee a fresh top slot for `v` holding a copy of the
    caller's value, and the matching pop re-exposes the caller's slot, which
    nothing above it can touch. When no activation of v's function reads `v`
    before writing it (a must-defined analysis over that function's blocks,
    parameters defined by the call block, a call that does not save `v` and
    may re-enter the function clobbering it) and the call block itself does
    not read `v` after the push, the copy is unobservable: the push only has
    to allocate the slot (device opcode `alloc`). Returns (block, op) positions.
    """
    fn_of = [lbl.split(".", 1)[0] for lbl in labels]
    n = len(flat.blocks)
    stacked = {v for v, c in classes.items() if c == "stacked"}
    vfn = {v: v.split(".", 1)[0] for v in stacked}
    calls: dict[str, set[str]] = {}
    callers: dict[int, list[int]] = {}
    for bi, b in enumerate(flat.blocks):
        if isinstance(b.terminator, ir.PushJump):
            calls.setdefault(fn_of[bi], set()).add(fn_of[b.terminator.jump_to])
            callers.setdefault(b.terminator.jump_to, []).append(bi)

    def reaches(g: str, f: str) -> bool:
        seen, todo = set(), [g]
        while todo:
            h = todo.pop()
            if h == f:
                return True
            if h not in seen:
                seen.add(h)
                todo.extend(calls.get(h, ()))
        return False

    def pushed_in(b: int) -> set[str]:
        return {op.output for op in flat.blocks[b].ops if isinstance(op, ir.Push)}

    exposed: set[str] = set()
    for f in set(fn_of):
        tracked = {v for v in stacked if vfn[v] == f}
        if not tracked:
            continue
        entries = [e for e in callers if fn_of[e] == f]
        if flat.entry < n and fn_of[flat.entry] == f and flat.entry not in entries:
            entries.append(flat.entry)
        state: dict[int, set[str]] = {}
        work = []
        for e in entries:
            if e == flat.entry and not callers.get(e):
                d = tracked & set(flat.inputs)
            else:  # parameters: written by every call block after its saves
                d = None
                for c in callers.get(e, ()):
                    w = {op.output for op in flat.blocks[c].ops
                         if isinstance(op, ir.Update) and op.output in tracked}
                    d = w if d is None else d & w
                d = d or set()
            state[e] = d if e not in state else state[e] & d
            work.append(e)
        while work:
            b = work.pop()
            blk = flat.blocks[b]
            d = set(state[b])
            ret_of = [c for c in range(n) if isinstance(flat.blocks[c].terminator, ir.PushJump)
                      and flat.blocks[c].terminator.return_to == b]
            saved_before = set.intersection(*(pushed_in(c) for c in ret_of)) if ret_of else set()
            for op in blk.ops:
                if isinstance(op, ir.Pop):
                    if op.var in tracked and op.var not in saved_before:
                        d.discard(op.var)
                    continue
                exposed.update(v for v in op.inputs if v in tracked and v not in d)
                if op.output in tracked:
                    d.add(op.output)
            t = blk.terminator
            succ: list[tuple[int, set[str]]] = []
            if isinstance(t, ir.FlatBranch):
                if t.cond in tracked and t.cond not in d:
                    exposed.add(t.cond)
                succ = [(t.true_target, d), (t.false_target, d)]
            elif isinstance(t, ir.FlatJump):
                succ = [(t.target, d)]
            elif isinstance(t, ir.PushJump):
                nd = d if not reaches(fn_of[t.jump_to], f) else d & pushed_in(b)
                succ = [(t.return_to, nd)]
            for s, sd in succ:
                if not (0 <= s < n) or fn_of[s] != f:
                    continue
                new = set(sd) if s not in state else state[s] & sd
                if s not in state or new != state[s]:
                    state[s] = new
                    work.append(s)
    out: set[tuple[int, int]] = set()
    for bi, blk in enumerate(flat.blocks):
        if not isinstance(blk.terminator, ir.PushJump):
            continue
        for oi, op in enumerate(blk.ops):
            if not (isinstance(op, ir.Push) and op.prim.name == "id" and op.inputs == (op.output,)):
                continue
            v = op.output
            if v not in stacked or v in exposed:
                continue
            if any(not isinstance(o, ir.Pop) and v in o.inputs for o in blk.ops[oi + 1:]):
                continue
            out.add((bi, oi))
    return out


def _op_liveness(flat: ir.FlatProgram):
    """live-after sets per (block, op index) of the flat program (Pop reads and writes)."""
    from .compiler import flat_live_in

    live_in = flat_live_in(flat)
    after: dict[tuple[int, int], set[str]] = {}
    n = len(flat.blocks)
    for bi, blk in enumerate(flat.blocks):
        live: set[str] = set()
        for s in ir.flat_successors(blk.terminator):
            if 0 <= s < n:
                live |= live_in[s]
        if isinstance(blk.terminator, ir.FlatBranch):
            live.add(blk.terminator.cond)
        for oi in range(len(blk.ops) - 1, -1, -1):
            op = blk.ops[oi]
            after[(bi, oi)] = set(live)
            if isinstance(op, ir.Pop):
                live.add(op.var)
            else:
                live.discard(op.output)
                live |= set(op.inputs)
    return after


def coalesce_copies(flat: ir.FlatProgram, classes: dict[str, str]) -> ir.FlatProgram:
    """Register copy coalescing: `update T = id R` with T defined only there and R
    never redefined while T is live gives T == R over T's whole life, so T can be
    renamed to R and the copy dropped (e.g. `build_tree.t1 = id build_tree._ret`)."""
    keep = set(flat.inputs) | {flat.output}
    defs: dict[str, list[tuple[int, int]]] = {}
    for bi, blk in enumerate(flat.blocks):
        for oi, op in enumerate(blk.ops):
            if not isinstance(op, ir.Pop):
                defs.setdefault(op.output, []).append((bi, oi))
    after = _op_liveness(flat)
    rename: dict[str, str] = {}

    def rep(v):
        while v in rename:
            v = rename[v]
        return v

    for bi, blk in enumerate(flat.blocks):
        for oi, op in enumerate(blk.ops):
            if not (isinstance(op, ir.Update) and op.prim.name == "id"):
                continue
            t, r = op.output, op.inputs[0]
            if t == r or t in keep or classes.get(t) != "register" or classes.get(r) != "register":
                continue
            if t in rename:
                continue
            # every definition of t must be a copy of the same r
            if any(not (isinstance(flat.blocks[db].ops[do], ir.Update)
                        and flat.blocks[db].ops[do].prim.name == "id"
                        and flat.blocks[db].ops[do].inputs == (r,))
                   for db, do in defs.get(t, ())):
                continue
            copies = set(defs.get(t, ()))
            root = rep(r)
            members = [root] + [v for v in rename if rep(v) == root]
            ok = True
            for m in members:
                for (db, do) in defs.get(m, ()):
                    if (db, do) in copies:
                        continue
                    if t in after[(db, do)]:
                        ok = False
                        break
                if not ok:
                    break
            # t's own uses must not overlap a live interval of another class member
            # that differs from r: only r's value flows into t, so the check above suffices
            if ok:
                rename[t] = r
                defs.setdefault(root, []).extend(defs.get(t, ()))
    if not rename:
        return flat

    def sub(v):
        return rep(v)

    blocks = []
    for blk in flat.blocks:
        ops = []
        for op in blk.ops:
            if isinstance(op, ir.Pop):
                ops.append(ir.Pop(sub(op.var)))
                continue
            out, ins = sub(op.output), tuple(sub(v) for v in op.inputs)
            if isinstance(op, ir.Update) and op.prim.name == "id" and ins == (out,):
                continue  # the coalesced copy itself (a Push of v = id v is a real save)
            ops.append(type(op)(out, op.prim, ins))
        t = blk.terminator
        if isinstance(t, ir.FlatBranch):
            t = ir.FlatBranch(sub(t.cond), t.true_target, t.false_target)
        blocks.append(ir.FlatBlock(tuple(ops), t))
    return ir.FlatProgram(tuple(blocks), flat.inputs, flat.output, flat.entry)


def forward_copies(flat: ir.FlatProgram, classes: dict[str, str]) -> ir.FlatProgram:
    """Copy forwarding through single-use temporaries: `update T = id X; ...; update V = id T`
    (T a temporary read only there) becomes `update V = id X` at T's position when nothing in
    between reads or writes V, and disappears when V is X. E.g. the argument copies of
    every call (`$a = id qp; ...; build_tree.q = id $a`): one copy instead of two, and
    none at all for a recursive call passing its own parameter (`q = id q`)."""
    blocks = []
    changed = False
    for blk in flat.blocks:
        ops = list(blk.ops)
        cond = blk.terminator.cond if isinstance(blk.terminator, ir.FlatBranch) else None
        uses: dict[str, list[int]] = {}
        defs: dict[str, list[int]] = {}
        for k, op in enumerate(ops):
            if isinstance(op, ir.Pop):
                continue
            for v in op.inputs:
                uses.setdefault(v, []).append(k)
            defs.setdefault(op.output, []).append(k)
        drop: set[int] = set()
        put: dict[int, object] = {}
        for k2, op in enumerate(ops):
            if not (isinstance(op, ir.Update) and op.prim.name == "id") or k2 in drop:
                continue
            t, v = op.inputs[0], op.output
            if classes.get(t) != "temporary" or t == v or t == cond or uses.get(t) != [k2]:
                continue
            if len(defs.get(t, ())) != 1:
                continue
            k1 = defs[t][0]
            src = ops[k1]
            if k1 >= k2 or k1 in drop or k1 in put or not (isinstance(src, ir.Update) and src.prim.name == "id"):
                continue
            x = src.inputs[0]
            between = ops[k1 + 1:k2]
            if any((isinstance(o, ir.Pop) and o.var == v) or
                   (not isinstance(o, ir.Pop) and (o.output == v or v in o.inputs)) for o in between):
                continue
            drop.add(k2)
            if x == v:
                drop.add(k1)
            else:
                put[k1] = ir.Update(v, src.prim, (x,))
            changed = True
        new_ops = [put.get(k, op) for k, op in enumerate(ops) if k not in drop]
        blocks.append(ir.FlatBlock(tuple(new_ops), blk.terminator))
    if not changed:
        return flat
    return ir.FlatProgram(tuple(blocks), flat.inputs, flat.output, flat.entry)


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


# ---- superblocks ---------------------------------------------------------------------------


def _is(op, out_cls, prim, ins=None):
    if not isinstance(op, ir.Update) or op.prim.name != prim and not prim.endswith("*"):
        return False
    if prim.endswith("*") and not op.prim.name.startswith(prim[:-1]):
        return False
    return ins is None or tuple(op.inputs) == tuple(ins)


def match_leapfrog(flat: ir.FlatProgram, classes: dict[str, str], grads: frozenset[str]) -> list[dict]:
    """Find leapfrog functions of the NUTS-lite program (reference workloads.py:461-472).

    Pattern, after demote_nonreentrant + fuse_copies (block indices b..b+3):
      b  : i = const:i64:0                                   jump b+1
      b+1: T1 = const:i64:L; T0 = lt i T1                    branch T0 b+2 b+3
      b+2: g = grad q; T3 = 2.0; T2 = div e T3; p = axpy T2 g p; q = axpy e p q;
           g = grad q; T5 = 2.0; T4 = div e T5; p = axpy T4 g p; T6 = 1; i = add i T6
                                                             jump b+1
      b+3: R = vcat q p                                      return
    with q, p, e, i, R registers, and b+1..b+3 entered only from inside.
    """
    found = []
    n = len(flat.blocks)
    preds = [[] for _ in range(n + 1)]
    for bi, blk in enumerate(flat.blocks):
        for s in ir.flat_successors(blk.terminator):
            preds[s].append(bi)
    for b in range(n - 3):
        b0, b1, b2, b3 = flat.blocks[b:b + 4]
        try:
            (o_i,) = b0.ops
            if not (_is(o_i, None, "const:i64:0") and isinstance(b0.terminator, ir.FlatJump)
                    and b0.terminator.target == b + 1):
                continue
            i = o_i.output
            t1, t0 = b1.ops
            if not (t1.prim.name.startswith("const:i64:") and _is(t0, None, "lt", (i, t1.output))):
                continue
            steps = int(t1.prim.name.split(":")[2])
            tb = b1.terminator
            if not (isinstance(tb, ir.FlatBranch) and tb.cond == t0.output
                    and (tb.true_target, tb.false_target) == (b + 2, b + 3)):
                continue
            ops = b2.ops
            if len(ops) != 11 or not (isinstance(b2.terminator, ir.FlatJump) and b2.terminator.target == b + 1):
                continue
            g1, c3, d2, ap1, aq, g2, c5, d4, ap2, c6, inc = ops
            gname = g1.prim.name
            q, gv = g1.inputs[0], g1.output
            if gname not in grads or g2.prim.name != gname or g2.inputs != (q,) or g2.output != gv:
                continue
            p = ap1.output
            e = d2.inputs[0]
            ok = (c3.prim.name == "const:f64:2.0" and _is(d2, None, "div", (e, c3.output))
                  and _is(ap1, None, "axpy", (d2.output, gv, p)) and _is(aq, None, "axpy", (e, p, q))
                  and aq.output == q and c5.prim.name == "const:f64:2.0"
                  and _is(d4, None, "div", (e, c5.output)) and _is(ap2, None, "axpy", (d4.output, gv, p))
                  and ap2.output == p and c6.prim.name == "const:i64:1"
                  and _is(inc, None, "add", (i, c6.output)) and inc.output == i)
            if not ok:
                continue
            (r,) = b3.ops
            if not (_is(r, None, "vcat", (q, p)) and isinstance(b3.terminator, ir.FlatReturn)):
                continue
            if any(classes.get(v) != "register" for v in (q, p, e, i, r.output)):
                continue
            if sorted(preds[b + 1]) != sorted([b, b + 2]) or preds[b + 2] != [b + 1] or preds[b + 3] != [b + 1]:
                continue
        except (ValueError, AttributeError, IndexError):
            continue
        found.append(dict(entry=b, head=b + 1, q=q, p=p, e=e, g=gv, i=i, ret=r.output,
                          steps=steps, grad=gname))
    return found


def _const_f64(op) -> float | None:
    if isinstance(op, ir.Update) and op.prim.name.startswith("const:f64:") and not op.inputs:
        return float(op.prim.name.split(":", 2)[2])
    return None


def match_normals(flat: ir.FlatProgram, classes: dict[str, str], labels) -> list[dict]:
    """Find Box-Muller momentum draws of the NUTS-lite program (reference
    workloads.py draw_normals; our workloads._normals emits the same text).

    One block ending in a return whose ops are, for pr = 0 .. P-1 (a = 2pr, b = a+1):
        Ta = const a; Xa = add c Ta; ua = rng_uniform key Xa      (same for b -> ub)
        r = sqrt(sub(0.0, mul(2.0, log(sub(1.0, ua)))))
        za = mul r (cos (mul 2pi ub));  [zb = mul r (sin (mul 2pi ub))  if b < k]
    then the left-to-right vcat of vfill:1(z0 .. z_{k-1}) and vfill:1(c + 2P) into
    the returned register. Every intermediate is a block-local temporary.
    """
    two_pi = 6.283185307179586
    found = []
    fn_of = [lbl.split(".", 1)[0] for lbl in labels]
    entries = {b.terminator.jump_to for b in flat.blocks if isinstance(b.terminator, ir.PushJump)}
    for b in sorted(entries):
        blk = flat.blocks[b]
        if not isinstance(blk.terminator, ir.FlatReturn):
            continue
        ops = blk.ops
        if any(not isinstance(o, ir.Update) for o in ops):
            continue
        pos = 0

        def take(prim, n_in=None):
            nonlocal pos
            if pos >= len(ops):
                raise ValueError
            o = ops[pos]
            if o.prim.name != prim or (n_in is not None and len(o.inputs) != n_in):
                raise ValueError
            pos += 1
            return o

        def take_const(value):
            nonlocal pos
            if pos >= len(ops) or _const_f64(ops[pos]) != value:
                raise ValueError
            pos += 1
            return ops[pos - 1].output

        try:
            key = c = None
            zs: list[str] = []
            pr = 0
            while pos < len(ops) and ops[pos].prim.name.startswith("const:f64:") and \
                    _const_f64(ops[pos]) == float(2 * pr) and pos + 1 < len(ops) and \
                    ops[pos + 1].prim.name == "add":
                us = []
                for off in (0, 1):
                    t = take_const(float(2 * pr + off))
                    x = take("add", 2)
                    if c is None:
                        c = x.inputs[0]
                    if x.inputs != (c, t):
                        raise ValueError
                    u = take("rng_uniform", 2)
                    if key is None:
                        key = u.inputs[0]
                    if u.inputs != (key, x.output):
                        raise ValueError
                    us.append(u.output)
                ua, ub = us
                t0, t2, t1 = take_const(0.0), take_const(2.0), take_const(1.0)
                s1 = take("sub", 2)
                lg = take("log", 1)
                m2 = take("mul", 2)
                s0 = take("sub", 2)
                r = take("sqrt", 1)
                if not (s1.inputs == (t1, ua) and lg.inputs == (s1.output,) and m2.inputs == (t2, lg.output)
                        and s0.inputs == (t0, m2.output) and r.inputs == (s0.output,)):
                    raise ValueError
                for trig in ("cos", "sin"):
                    if trig == "sin" and (pos >= len(ops) or _const_f64(ops[pos]) != two_pi):
                        break
                    tp = take_const(two_pi)
                    mu = take("mul", 2)
                    tr = take(trig, 1)
                    z = take("mul", 2)
                    if not (mu.inputs == (tp, ub) and tr.inputs == (mu.output,) and z.inputs == (r.output, tr.output)):
                        raise ValueError
                    zs.append(z.output)
                pr += 1
            k, pairs = len(zs), pr
            if pairs == 0 or not (2 * pairs - 1 <= k <= 2 * pairs) or c is None:
                raise ValueError
            # pack: vfill:1 of each z, chained left to right, then vfill:1(c + 2P)
            acc = None
            for i, z in enumerate(zs):
                f = take("vfill:1", 1)
                if f.inputs != (z,):
                    raise ValueError
                if acc is None:
                    acc = f.output
                    continue
                v = take("vcat", 2)
                if v.inputs != (acc, f.output):
                    raise ValueError
                acc = v.output
            tc = take_const(float(2 * pairs))
            xc = take("add", 2)
            fc = take("vfill:1", 1)
            ret = take("vcat", 2)
            if xc.inputs != (c, tc) or fc.inputs != (xc.output,) or ret.inputs != (acc, fc.output):
                raise ValueError
            if pos != len(ops) or classes.get(ret.output) != "register":
                raise ValueError
        except (ValueError, AttributeError, IndexError):
            continue
        found.append(dict(entry=b, key=key, c=c, ret=ret.output, k=k, pairs=pairs))
    return found


def superblock_io(flat: ir.FlatProgram, m: dict, classes: dict | None = None) -> tuple[dict, set[tuple[int, int]], int, list]:
    """Operand forwarding and dead side outputs of a fused leapfrog function `m`.

    The superblock runs immediately after its call block, so an argument copied
    there as `A = id X; leapfrog.q = id A` (A a temporary used only for that)
    can be read from X's current top by the superblock itself: both copies go
    (X must not be written, pushed or popped later in the call block). The
    function's locals q, p, g, i are written back only when some block outside
    the function reads them. Returns ({param: source}, dropped (block, op)
    positions, writeback flag for q/p, [g or None, i or None]).
    """
    body = {m["entry"], m["entry"] + 1, m["entry"] + 2, m["entry"] + 3}

    def read_outside(v):
        for bi, blk in enumerate(flat.blocks):
            if bi in body:
                continue
            if isinstance(blk.terminator, ir.FlatBranch) and blk.terminator.cond == v:
                return True
            if any(not isinstance(o, ir.Pop) and v in o.inputs for o in blk.ops):
                return True
        return False

    callers = [bi for bi, blk in enumerate(flat.blocks)
               if isinstance(blk.terminator, ir.PushJump) and blk.terminator.jump_to == m["entry"]]
    fwd, drop = {}, set()
    for param in (m["q"], m["p"]):
        # the program's entry function is also entered without a call: its parameters are
        # the inputs, never a caller's argument sources
        if read_outside(param) or not callers or m["entry"] == flat.entry:
            continue
        srcs, pos = set(), set()
        for cb in callers:
            ops = flat.blocks[cb].ops
            defs = [k for k, o in enumerate(ops) if not isinstance(o, ir.Pop) and o.output == param]
            if len(defs) != 1:
                break
            k = defs[0]
            o = ops[k]
            if not (isinstance(o, ir.Update) and o.prim.name == "id"):
                break
            a = o.inputs[0]
            adefs = [j for j, x in enumerate(ops[:k]) if not isinstance(x, ir.Pop) and x.output == a]
            uses = [j for j, x in enumerate(ops) if not isinstance(x, ir.Pop) and a in x.inputs]
            ad = ops[adefs[0]] if len(adefs) == 1 else None
            if (uses == [k] and a.split(".", 1)[-1].startswith("$a") and isinstance(ad, ir.Update)
                    and ad.prim.name == "id"):
                x, start, here = ad.inputs[0], adefs[0], {(cb, adefs[0]), (cb, k)}
            elif (classes or {}).get(a, "temporary") != "temporary":  # param = id X (forward_copies)
                x, start, here = a, k, {(cb, k)}
            else:
                break
            if any((isinstance(y, ir.Pop) and y.var == x) or (not isinstance(y, ir.Pop) and y.output == x)
                   for y in ops[start + 1:]):
                break
            srcs.add(x)
            pos |= here
        else:
            if len(srcs) == 1:
                fwd[param] = srcs.pop()
                drop |= pos
    writeback = int(read_outside(m["q"]) or read_outside(m["p"]))
    refs = [m["g"] if read_outside(m["g"]) else None, m["i"] if read_outside(m["i"]) else None]
    return fwd, drop, writeback, refs


def fuse_leaf_logpdf(flat: ir.FlatProgram, m: dict, logpdf_name: str, dim: int) -> tuple[int, int] | None:
    """The caller's `logpdf(q1)` right after a fused leapfrog returns.

    In NUTS-lite's leaf (reference workloads.py:388-396) the only call site's
    return block evaluates `logpdf(vslice:0:d(leapfrog(...)))`: the log density
    at the final position, whose contraction q.(P q) the superblock's last kick
    has just formed. The superblock then also writes the fast logpdf (same DMMA
    accumulators, same fma order as warp_gauss) to a register the logpdf op
    reads when `exact_logpdf` is off. Returns (block, op) of that logpdf op.
    """
    callers = [bi for bi, blk in enumerate(flat.blocks)
               if isinstance(blk.terminator, ir.PushJump) and blk.terminator.jump_to == m["entry"]]
    rets = {flat.blocks[c].terminator.return_to for c in callers}
    if len(rets) != 1:
        return None
    rb = rets.pop()
    alias, views = {m["ret"]}, set()
    for k, o in enumerate(flat.blocks[rb].ops):
        if isinstance(o, ir.Pop):
            if o.var in alias | views:
                return None
            continue
        if o.prim.name == logpdf_name and len(o.inputs) == 1 and o.inputs[0] in views:
            return rb, k
        if o.prim.name == "id" and o.inputs[0] in alias and o.output not in alias | views:
            alias.add(o.output)
        elif o.prim.name == f"vslice:0:{dim}" and o.inputs[0] in alias and o.output not in alias | views:
            views.add(o.output)
        elif o.output in alias | views:
            return None
    return None


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
    flat_rows: int = 0                                     # per-lane rows of non-stacked storage


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


def _storage(block_ops: list[list[dict]], conds: list[str | None], classes: dict[str, str],
             vtype, keep: set[str], optimize: bool):
    """Assign every operand a device variable and every device variable its rows.

    Returns (var list [(name, cls, VType, row)], renamed block_ops, renamed conds,
    flat_rows). Rows of stacked variables are assigned by the C library after
    the flat region (they depend on the machine's stack depth).

    optimize=False: one device variable per program variable, private rows.
    optimize=True: temporaries (block-local by construction, compiler.py:421-479)
    are renamed per definition, then
      * `T = id S` / `T = vslice:lo:hi S` with S at a static location that is not
        rewritten while T lives becomes a zero-copy view of S's rows;
      * `T = vcat(A, X)` where A (a temporary owning its rows) dies at this op
        extends A in place (the VM skips the copy when dst == A);
      * remaining temporaries share one per-lane arena by interval colouring.
    """
    entries: list[list] = []   # [name, cls, VType, row]
    index: dict[str, int] = {}

    def add(name, cls, vt, row=-1):
        index[name] = len(entries)
        entries.append([name, cls, vt, row])
        return index[name]

    flat_rows = 0
    persistent = sorted(v for v, c in classes.items() if c != "temporary" or v in keep or not optimize)
    for v in persistent:
        cls = classes.get(v, "temporary")
        vt = vtype(v)
        if cls == "stacked":
            add(v, cls, vt)
        else:
            add(v, cls, vt, flat_rows)
            flat_rows += words(vt)
    if not optimize:
        renamed = [[dict(op, out=index[op["out"]], ins=[index[i] for i in op["ins"]]) for op in ops]
                   for ops in block_ops]
        return entries, renamed, [index[c] if c else 0 for c in conds], flat_rows

    is_temp = {v for v, c in classes.items() if c == "temporary" and v not in keep}
    arena_base = flat_rows
    arena_size = 0
    new_blocks, new_conds = [], []
    for bi, ops in enumerate(block_ops):
        # --- SSA-rename temporaries of this block
        cur: dict[str, str] = {}
        inst: dict[str, dict] = {}   # instance -> info
        renamed = []
        for k, op in enumerate(ops):
            ins = [cur.get(i, i) for i in op["ins"]]
            for i in ins:
                if i in inst:
                    inst[i]["end"] = max(inst[i]["end"], k)
            out = op["out"]
            if out in is_temp and op["action"] != ACTION_POP:
                name = f"{out}@{bi}.{k}"
                cur[out] = name
                inst[name] = {"start": k, "end": k, "vt": vtype(out), "op": k}
                out = name
            renamed.append(dict(op, out=out, ins=ins))
        cond = conds[bi]
        if cond is not None:
            cond = cur.get(cond, cond)
            if cond in inst:
                inst[cond]["end"] = max(inst[cond]["end"], len(ops))

        # registers written inside this block, by op position
        writes: dict[str, list[int]] = {}
        for k, op in enumerate(renamed):
            if op["out"] not in inst:
                writes.setdefault(op["out"], []).append(k)

        def stable(src: str, a: int, b: int) -> bool:
            """src keeps its value and location over ops (a, b]."""
            if src in inst:
                return True
            if classes.get(src) != "register" and src not in keep:
                return False
            return not any(a < w <= b for w in writes.get(src, ()))

        # --- views and in-place vcat chains
        owner: dict[str, tuple[str, int]] = {}   # instance -> (root owner, word offset)
        chained: set[str] = set()                # instances that extend a vcat chain in place

        def root(n):
            return owner.get(n, (n, 0))

        for name, info in sorted(inst.items(), key=lambda kv: kv[1]["start"]):
            op = renamed[info["op"]]
            prim, end = op["prim"], info["end"]
            if prim == "id" or prim.startswith("vslice:"):
                src = op["ins"][0]
                lo = int(prim.split(":")[1]) if prim != "id" else 0
                if (src in inst or classes.get(src) == "register" or src in keep) \
                        and classes.get(src) != "stacked" and stable(src, info["start"], end):
                    r, off = root(src)
                    owner[name] = (r, off + lo)
                    if r in inst:
                        inst[r]["end"] = max(inst[r]["end"], end)
            elif prim == "vcat":
                a = op["ins"][0]
                # extend a's storage in place when a dies here and owns its rows (or is
                # itself a chain member at offset 0 of a temporary's rows)
                head = a
                while head in owner and owner[head][1] == 0 and head in chained:
                    head = owner[head][0]
                if a in inst and (a not in owner or a in chained) and head in inst \
                        and head not in owner and inst[a]["end"] == info["start"] \
                        and op["ins"][1] != a and root(op["ins"][1])[0] not in (a, head):
                    owner[name] = (head, 0)
                    chained.add(name)
                    inst[head]["end"] = max(inst[head]["end"], end)
                    inst[head]["span"] = max(inst[head].get("span", words(inst[head]["vt"])),
                                             words(info["vt"]))
        # the storage owner of every view / chain member must outlive it
        for name in owner:
            r = name
            while r in owner:
                r = owner[r][0]
            if r in inst:
                inst[r]["end"] = max(inst[r]["end"], inst[name]["end"])

        # --- chain sinks: a vcat chain whose last link writes a register V (that no
        # other op of the chain's lifetime touches) is built directly in V's rows,
        # so the final copy disappears (e.g. NUTS-lite's leaf/node packs into _ret)
        sinks: dict[str, int] = {}
        for k, op in enumerate(renamed):
            v = op["out"]
            if op["prim"] != "vcat" or v in inst or classes.get(v) != "register" or v not in index:
                continue
            a = op["ins"][0]
            if a not in inst:
                continue
            r, off = a, 0
            while r in owner:
                off += owner[r][1]
                r = owner[r][0]
            if off != 0 or r not in inst or r in sinks or inst[r]["end"] != k:
                continue
            if any(v == o["out"] or v in o["ins"] for o in renamed[inst[r]["start"]:k]):
                continue
            if op["ins"][1] == v or root(op["ins"][1])[0] == r:
                continue
            sinks[r] = entries[index[v]][3]

        # --- arena allocation (first fit by start, closed intervals)
        live: list[tuple[int, int, int]] = []  # (end, offset, size)
        top = 0
        placed: dict[str, int] = {}
        for name, info in sorted(inst.items(), key=lambda kv: (kv[1]["start"], kv[0])):
            if name in sinks:
                continue
            if name in owner:
                continue
            size = info.get("span", words(info["vt"]))
            live = [x for x in live if x[0] >= info["start"]]
            off, ok = 0, False
            for cand in sorted({0} | {o + s for _, o, s in live}):
                if all(cand + size <= o or cand >= o + s for _, o, s in live):
                    off, ok = cand, True
                    break
            assert ok
            placed[name] = off
            live.append((info["end"], off, size))
            top = max(top, off + size)
        arena_size = max(arena_size, top)

        def final_row(n):
            r, off = n, 0
            while r in owner:
                r2, o2 = owner[r]
                off += o2
                r = r2
            if r in placed:
                return arena_base + placed[r] + off
            if r in sinks:
                return sinks[r] + off
            return entries[index[r]][3] + off

        for name, info in inst.items():
            add(name, "temporary", info["vt"], final_row(name))
        out_ops = []
        for op in renamed:
            d = dict(op, out=index[op["out"]], ins=[index[i] for i in op["ins"]])
            if "refs" in op:  # superblock side outputs; dead temporaries are skipped (-1)
                d["refs"] = [-1 if (r is None or r in is_temp) else index[r] for r in op["refs"]]
            for key in ("lp", "cache"):  # fused leaf logpdf register
                if key in op:
                    d[key] = index[op[key]]
            out_ops.append(d)
        new_blocks.append(out_ops)
        new_conds.append(index[cond] if cond is not None else 0)
    return entries, new_blocks, new_conds, arena_base + arena_size


def lower(compiled: CompiledProgram, types: dict[str, VType], *, optimize: bool = True,
          superblocks: bool = False, max_superblock_dim: int = 256) -> DeviceProgram:
    """Build the device tables for `compiled` given inferred lane types.

    superblocks=True (warp-group engine only) replaces each recognised
    leapfrog function entry with one fused LS_OP_LEAPFROG op + return.
    """
    flat, classes = compiled.flat, dict(compiled.classes)
    allocs: set[tuple[int, int]] = set()
    if optimize:
        flat, classes = demote_nonreentrant(flat, classes, compiled.labels)
        flat, classes = demote_unpushed(flat, classes)
        flat = fuse_copies(flat, classes)
        flat = forward_copies(flat, classes)
        flat = coalesce_copies(flat, classes)
        allocs = dead_saves(flat, classes, compiled.labels)
    normals = {}
    if optimize:
        for m in match_normals(flat, classes, compiled.labels):
            if types.get(m["c"], VType("i64")).kind == "f64" and types.get(m["ret"]) is not None \
                    and words(types[m["ret"]]) == m["k"] + 1:
                normals[m["entry"]] = m
    fused = {}
    if optimize and superblocks:
        for m in match_leapfrog(flat, classes, grad_names()):
            t = device_op(m["grad"]).target
            if t is not None and t.kind == 1 and t.dim <= max_superblock_dim:
                fused[m["entry"]] = m
    dropped: set[tuple[int, int]] = set()
    cached_logpdf: dict[tuple[int, int], str] = {}
    for m in fused.values():
        m["fwd"], drop, m["writeback"], m["live_refs"] = superblock_io(flat, m, classes)
        dropped |= drop
        t = device_op(m["grad"]).target
        lp_name = next((tt.logpdf for tt in _registered() if tt.grad == m["grad"]), None)
        hit = fuse_leaf_logpdf(flat, m, lp_name, t.dim) if lp_name and (t.dim + 7) // 8 <= 16 else None
        m["lp"] = None
        if hit is not None:
            m["lp"] = m["ret"].split(".", 1)[0] + ".$lp"
            classes[m["lp"]] = "register"
            cached_logpdf[hit] = m["lp"]

    grads = grad_names()
    for n in set(types):
        classes.setdefault(n, "temporary")
    extra_types: dict[str, VType] = {}
    for m in fused.values():
        if m.get("lp"):
            extra_types[m["lp"]] = VType("f64")

    def vtype(v: str) -> VType:
        return extra_types.get(v) or types.get(v, VType("i64"))

    targets: list = []
    ref_prims = _block_prims(compiled.flat)
    block_ops: list[list[dict]] = []
    conds: list[str | None] = []
    terms = []
    n_scratch = 0
    for bi, blk in enumerate(flat.blocks):
        ops: list[dict] = []
        if bi in fused:
            m = fused[bi]
            t = device_op(m["grad"]).target
            if t not in targets:
                targets.append(t)
            # kind bit 0: write the final q, p back to the function's registers
            ops.append(dict(opcode=OPCODES["leapfrog"], action=ACTION_UPDATE, out=m["ret"],
                            ins=[m["fwd"].get(m["q"], m["q"]), m["fwd"].get(m["p"], m["p"]), m["e"]],
                            kind=m["writeback"], width=2 * t.dim,
                            imm0=targets.index(t), imm1=m["steps"], imm2=m["head"], bits=0,
                            prim="$leapfrog", refs=m["live_refs"], **({"lp": m["lp"]} if m["lp"] else {})))
            terms.append((TERM_RETURN, 0, 0))
            conds.append(None)
            block_ops.append(ops)
            continue
        if bi in normals:
            m = normals[bi]
            ops.append(dict(opcode=OPCODES["normals"], action=ACTION_UPDATE, out=m["ret"], ins=[m["key"], m["c"]],
                            kind=KIND_CODE[vtype(m["key"]).kind], width=m["k"] + 1, imm0=m["k"],
                            imm1=m["pairs"], imm2=0, bits=0, prim="$normals"))
            terms.append((TERM_RETURN, 0, 0))
            conds.append(None)
            block_ops.append(ops)
            continue
        for oi, op in enumerate(blk.ops):
            if isinstance(op, ir.Pop):
                ops.append(dict(opcode=0, action=ACTION_POP, out=op.var, ins=[], kind=0, width=1,
                                imm0=0, imm1=0, imm2=0, bits=0, prim="$pop"))
                continue
            if (bi, oi) in dropped:  # argument copies forwarded into a superblock
                continue
            if (bi, oi) in allocs:
                vt = vtype(op.output)
                ops.append(dict(opcode=OPCODES["alloc"], action=ACTION_PUSH, out=op.output, ins=[],
                                kind=KIND_CODE[vt.kind], width=words(vt), imm0=0, imm1=0, imm2=0, bits=0,
                                prim="$alloc"))
                continue
            dev = device_op(op.prim.name)
            if dev is None:
                raise NotImplementedError(
                    f"primitive '{op.prim.name}' has no B200 implementation (host-only kernel); "
                    "the lockstep B200 engine has no CPU fallback")
            out_vt = vtype(op.output)
            in_kind = KIND_CODE[vtype(op.inputs[0]).kind] if op.inputs else KIND_CODE[out_vt.kind]
            imm0, imm1, bits = dev.imm0, dev.imm1, 0
            if dev.opcode == OPCODES["const"]:
                bits, imm0 = dev.imm0, 0
            if dev.target is not None:
                if dev.target not in targets:
                    targets.append(dev.target)
                imm0 = targets.index(dev.target)
            action = ACTION_PUSH if isinstance(op, ir.Push) else ACTION_UPDATE
            row = dict(opcode=dev.opcode, action=action, out=op.output, ins=list(op.inputs),
                       kind=in_kind, width=words(out_vt), imm0=imm0, imm1=imm1, imm2=0, bits=bits,
                       prim=op.prim.name)
            if (bi, oi) in cached_logpdf:  # written by the preceding superblock (fast mode)
                row["cache"] = cached_logpdf[(bi, oi)]
            if action == ACTION_UPDATE and op.output in op.inputs and not _inplace_safe(op, op.output):
                tmp = f"$scratch{n_scratch}"
                n_scratch += 1
                extra_types[tmp] = out_vt
                classes[tmp] = "temporary"
                ops.append(dict(row, out=tmp))
                ops.append(dict(opcode=OPCODES["id"], action=ACTION_UPDATE, out=op.output, ins=[tmp],
                                kind=KIND_CODE[out_vt.kind], width=words(out_vt), imm0=0, imm1=0,
                                imm2=0, bits=0, prim="id"))
            else:
                ops.append(row)
        t = blk.terminator
        if isinstance(t, ir.FlatJump):
            terms.append((TERM_JUMP, t.target, 0))
            conds.append(None)
        elif isinstance(t, ir.FlatBranch):
            terms.append((TERM_BRANCH, t.true_target, t.false_target))
            conds.append(t.cond)
        elif isinstance(t, ir.PushJump):
            terms.append((TERM_PUSHJUMP, t.jump_to, t.return_to))
            conds.append(None)
        else:
            terms.append((TERM_RETURN, 0, 0))
            conds.append(None)
        block_ops.append(ops)

    keep = set(flat.inputs) | {flat.output}
    entries, dev_blocks, dev_conds, flat_rows = _storage(block_ops, conds, classes, vtype, keep, optimize)

    op_rows, block_rows = [], []
    for bi, ops in enumerate(dev_blocks):
        begin = len(op_rows)
        for op in ops:
            ins = op["ins"] + [0] * (3 - len(op["ins"]))
            bits = op["bits"]
            if "refs" in op:  # superblock side outputs: g (or -1 when dead) | i << 32
                gref, iref = op["refs"]
                bits = (gref & 0xFFFFFFFF) | (iref << 32)
            kind = op["kind"]
            if "lp" in op:  # superblock: kind bit 0 = q/p write-back, kind >> 1 = lp var + 1
                kind |= (op["lp"] + 1) << 1
            if "cache" in op:  # logpdf: bits = cached value var + 1
                bits = op["cache"] + 1
            op_rows.append((op["opcode"], op["action"], op["out"], len(op["ins"]), ins, kind,
                            op["width"], op["imm0"], op["imm1"], op["imm2"], bits))
        g = sum(n for name, n in ref_prims[bi].items() if name in grads)
        if bi in fused:  # the superblock performs every gradient of the function's L iterations
            body = fused[bi]["entry"] + 2
            g = fused[bi]["steps"] * sum(n for name, n in ref_prims[body].items() if name in grads)
        tt = terms[bi]
        block_rows.append((begin, len(op_rows) - begin, tt[0], tt[1], tt[2], dev_conds[bi], g, 0))

    var_arr = np.zeros(len(entries), dtype=VAR_DTYPE)
    sp_row = 0
    for i, (name, cls, vt, row) in enumerate(entries):
        var_arr[i] = (CLASS_CODE[cls], KIND_CODE[vt.kind], words(vt),
                      sp_row if cls == "stacked" else -1, row, 0)
        if cls == "stacked":
            sp_row += 1
    ops_arr = np.zeros(len(op_rows), dtype=OP_DTYPE)
    for i, r in enumerate(op_rows):
        ops_arr[i] = r
    blocks = np.array(block_rows, dtype=BLOCK_DTYPE) if block_rows else np.zeros(0, BLOCK_DTYPE)
    names = [e[0] for e in entries]
    index = {n: i for i, n in enumerate(names)}
    return DeviceProgram(
        compiled=compiled, flat=flat, classes={e[0]: e[1] for e in entries},
        types={e[0]: e[2] for e in entries}, var_names=names, var_index=index, blocks=blocks,
        ops=ops_arr, vars=var_arr, inputs=np.array([index[v] for v in flat.inputs], dtype=np.int32),
        output=index[flat.output], targets=targets, block_prims=ref_prims,
        block_stack_ops=_block_stack_ops(compiled.flat, compiled.classes), optimized=optimize,
        flat_rows=flat_rows)
