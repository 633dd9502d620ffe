"""Block-selection rules of the B200 VM (which populated block runs next).

Per-lane results never depend on the rule (lane isolation, reference
PAPER.md:601-611, tests/test_local_exec.py:83-88); the global schedule, the
step count and the number of lanes that share each batched block execution
do. Keyed rules pick the least key among the blocks live lanes sit at; a key
carries its block index in bits 0..15 (include/lockstep_b200.h).

* ``min_pc`` — the reference rule (pc_vm.py:306-311): key = block index.
* ``most_populated`` — the paper's throughput heuristic (max live lanes).
* ``local`` — Alg. 1, the local-static engine (reference local_exec.py:81-185)
  executed on the flat program: the deepest activation runs until it returns,
  a call's landing pad runs first when it does (the call-graph block the call
  sat in completes), otherwise the lowest block of the activation.
* ``priority`` — reverse post-order over the interprocedural CFG (a block
  runs once every lane that can still reach it along forward edges has
  arrived), with blocks that hold target contractions (fused leapfrogs,
  gradients) and the exits of recursive functions deferred behind all others
  so they execute with as many lanes as possible.
"""

from __future__ import annotations

import numpy as np

from . import ir

SCHEDULES = ("min_pc", "most_populated", "local", "priority")
SCHED_CODE = {"min_pc": 0, "most_populated": 1, "local": 2, "priority": 3}


def _fn_of(labels) -> list[str]:
    return [lbl.split(".", 1)[0] for lbl in labels]


def _successors(flat: ir.FlatProgram, labels) -> dict[int, list[int]]:
    """Interprocedural successor lists: a call continues at its callee entry and (after the
    callee returns) at its landing pad; a return reaches every landing pad of its function."""
    n = len(flat.blocks)
    fn = _fn_of(labels)
    pads: dict[str, list[int]] = {}
    for blk in flat.blocks:
        t = blk.terminator
        if isinstance(t, ir.PushJump):
            pads.setdefault(fn[t.jump_to], []).append(t.return_to)
    succ: dict[int, list[int]] = {}
    for b, blk in enumerate(flat.blocks):
        t = blk.terminator
        if isinstance(t, ir.PushJump):
            succ[b] = [t.jump_to, t.return_to]
        elif isinstance(t, ir.FlatReturn):
            succ[b] = list(pads.get(fn[b], []))
        else:
            succ[b] = [s for s in ir.flat_successors(t) if 0 <= s < n]
    return succ


def reverse_post_order(flat: ir.FlatProgram, labels) -> list[int]:
    """Blocks in reverse post-order of a DFS from the entry; unreachable blocks last."""
    succ = _successors(flat, labels)
    seen: set[int] = set()
    post: list[int] = []
    stack = [(flat.entry, iter(succ.get(flat.entry, ())))]
    seen.add(flat.entry)
    while stack:
        u, it = stack[-1]
        for v in it:
            if v not in seen:
                seen.add(v)
                stack.append((v, iter(succ.get(v, ()))))
                break
        else:
            stack.pop()
            post.append(u)
    order = post[::-1]
    return order + [b for b in range(len(flat.blocks)) if b not in seen]


def recursive_functions(flat: ir.FlatProgram, labels) -> set[str]:
    fn = _fn_of(labels)
    calls: dict[str, set[str]] = {}
    for b, blk in enumerate(flat.blocks):
        if isinstance(blk.terminator, ir.PushJump):
            calls.setdefault(fn[b], set()).add(fn[blk.terminator.jump_to])
    out = set()
    for f in set(fn):
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


def landing_pads(flat: ir.FlatProgram) -> set[int]:
    return {blk.terminator.return_to for blk in flat.blocks if isinstance(blk.terminator, ir.PushJump)}


def block_keys(flat: ir.FlatProgram, labels, rule: str, contraction_blocks=()) -> np.ndarray:
    """uint32 key per block for the keyed rules (min_pc, local, priority)."""
    n = len(flat.blocks)
    if n >= 1 << 16:
        raise ValueError("keyed schedules support at most 65535 blocks")
    idx = np.arange(n, dtype=np.uint32)
    if rule in ("min_pc", "most_populated"):
        return idx
    if rule == "local":
        pads = landing_pads(flat)
        return np.array([(0 if b in pads else 1) << 16 | b for b in range(n)], dtype=np.uint32)
    if rule == "priority":
        rec = recursive_functions(flat, labels)
        fn = _fn_of(labels)
        deferred = set(int(b) for b in contraction_blocks)
        deferred |= {b for b, blk in enumerate(flat.blocks)
                     if isinstance(blk.terminator, ir.FlatReturn) and fn[b] in rec}
        order = reverse_post_order(flat, labels)
        rank = {b: r for r, b in enumerate(sorted(order, key=lambda b: (b in deferred, order.index(b))))}
        return np.array([(rank[b] << 16) | b for b in range(n)], dtype=np.uint32)
    raise ValueError(f"unknown schedule '{rule}' (one of {SCHEDULES})")


def select(rule: str, tops: np.ndarray, depths: np.ndarray, keys: np.ndarray, halt: int):
    """Host mirror of the device selection for a single group: (block, selected-lane mask).
    `tops` are the lanes' pcs, `depths` their pc-stack pointers."""
    live = tops != halt
    if not live.any():
        return halt, np.zeros_like(live)
    if rule == "most_populated":
        vals, counts = np.unique(tops[live], return_counts=True)
        b = int(vals[np.argmax(counts)])
        return b, live & (tops == b)
    k = keys[np.where(live, tops, 0)].astype(np.uint64)
    if rule == "local":
        d = np.clip(depths, 0, 255).astype(np.uint64)
        k = ((255 - d) << np.uint64(24)) | (k & np.uint64(0xFFFFFF))
    k = np.where(live, k, np.uint64(0xFFFFFFFFFFFF))
    best = k.min()
    sel = live & (k == best)
    return int(best & np.uint64(0xFFFF)), sel

