"""CPU simulator of the device program tables (test infrastructure only).

Executes a `lowering.DeviceProgram` one lane at a time over a per-lane
workspace laid out exactly like the CUDA VM's (csrc/vm.cu): non-stacked
variables at their lowered `row`, stacked variables after `flat_rows`, top
slot under the stack pointer. Because lanes are independent, running each
lane to completion is equivalent to any batched schedule.

Its purpose is to catch storage-assignment bugs (temporary arena sharing,
zero-copy views, in-place vcat chains, demoted stacks) on the CPU: the
tables must produce the oracle's results. Arithmetic uses numpy scalar
ops; target kernels reuse the oracle's numpy forms, so results match the
oracle to rounding, and integer/control results exactly.
"""

from __future__ import annotations

import numpy as np

from . import lockstep_oracle as O

OPN = {1: "const", 2: "id", 3: "add", 4: "sub", 5: "mul", 6: "div", 7: "min", 8: "max", 9: "le",
       10: "lt", 11: "eq", 12: "and", 13: "or", 14: "not", 15: "neg", 16: "abs", 17: "sqrt",
       18: "exp", 19: "log", 20: "sin", 21: "cos", 22: "floor", 23: "select", 24: "dot",
       25: "axpy", 26: "vget", 27: "vstore", 28: "vcat", 29: "vfill", 30: "vslice", 31: "rng_uniform",
       32: "logpdf", 33: "grad", 65: "alloc", 66: "normals"}


class Fault(Exception):
    pass


def _f(w):
    return np.uint64(w).view(np.float64)


def _w(x):
    return np.float64(x).view(np.uint64)


def run_lane(dp, inputs_words: list[np.ndarray], depth: int, max_steps: int = 10**7):
    """Run one lane; inputs_words[k] is the lane's input k as uint64 words."""
    vars_ = dp.vars
    nb = len(dp.blocks)
    rows = dp.flat_rows
    var_row = np.zeros(len(vars_), np.int64)
    for v in range(len(vars_)):
        if vars_[v]["cls"] == 0:
            var_row[v] = rows
            rows += depth * vars_[v]["width"]
        else:
            var_row[v] = vars_[v]["row"]
    ws = np.zeros(rows, np.uint64)
    n_sp = int(max(vars_["sp"].max(), -1)) + 1
    sp = np.ones(n_sp, np.int64)
    for k, v in enumerate(dp.inputs):
        w = int(vars_[v]["width"])
        ws[var_row[v]:var_row[v] + w] = inputs_words[k]
    pcs = [nb, dp.flat.entry]
    blocks_seen = []

    def top(v):
        if vars_[v]["cls"] == 0:
            s = max(sp[vars_[v]["sp"]] - 1, 0)
            return var_row[v] + s * vars_[v]["width"]
        return var_row[v]

    def vec(v):
        base = top(v)
        return ws[base:base + vars_[v]["width"]].copy()

    def as_i64(word, kind):
        return O.rng_uniform.__globals__["np"].int64(np.array([_f(word)]).astype(np.int64)[0]) \
            if kind == 0 else np.int64(np.uint64(word).view(np.int64))

    targets = dp.targets
    steps = 0
    while pcs[-1] != nb:
        b = pcs[-1]
        blocks_seen.append(b)
        blk = dp.blocks[b]
        for op in dp.ops[blk["op_begin"]:blk["op_begin"] + blk["op_count"]]:
            v = int(op["out"])
            if op["action"] == 2:
                if sp[vars_[v]["sp"]] < 1:
                    raise Fault(("underflow", v))
                sp[vars_[v]["sp"]] -= 1
                continue
            res = None if OPN[int(op["opcode"])] == "alloc" else _compute(op, vec, vars_, targets, as_i64)
            if vars_[v]["cls"] == 0:
                r = vars_[v]["sp"]
                if op["action"] == 0:
                    if sp[r] >= depth:
                        raise Fault(("overflow", v))
                    base = var_row[v] + sp[r] * vars_[v]["width"]
                    sp[r] += 1
                else:
                    if sp[r] < 1:
                        raise Fault(("underflow", v))
                    base = var_row[v] + (sp[r] - 1) * vars_[v]["width"]
            else:
                base = var_row[v]
            if res is not None:  # alloc: the new top slot is left as it was
                ws[base:base + len(res)] = res
        t = blk["term"]
        if t == 0:
            pcs[-1] = int(blk["a"])
        elif t == 1:
            pcs[-1] = int(blk["a"]) if ws[top(int(blk["cond"]))] != 0 else int(blk["b"])
        elif t == 2:
            pcs[-1] = int(blk["b"])
            if len(pcs) >= depth + 1:
                raise Fault(("overflow", -1))
            pcs.append(int(blk["a"]))
        else:
            pcs.pop()
        steps += 1
        if steps > max_steps:
            raise RuntimeError("step limit")
    return vec(dp.output), blocks_seen


def _compute(op, vec, vars_, targets, as_i64):
    name = OPN[int(op["opcode"])]
    ins = [int(i) for i in op["in"][:op["nin"]]]
    f = op["kind"] == 0
    if name == "const":
        return np.array([np.int64(op["bits"]).view(np.uint64)], np.uint64)
    xs = [vec(i) for i in ins]
    if name == "id":
        return xs[0]
    with np.errstate(all="ignore"):
        if name in ("add", "sub", "mul", "div", "min", "max"):
            dt = np.float64 if f else np.int64
            a, b = xs[0].view(dt), xs[1].view(dt)
            fn = O._BASE[name]
            return np.asarray(fn(a, b), dt).view(np.uint64)
        if name in ("le", "lt", "eq"):
            dt = np.float64 if f else np.int64
            return np.array([int(O._BASE[name](xs[0].view(dt)[0], xs[1].view(dt)[0]))], np.uint64)
        if name in ("and", "or"):
            return np.array([int(O._BASE[name](xs[0][0] != 0, xs[1][0] != 0))], np.uint64)
        if name == "not":
            return np.array([int(xs[0][0] == 0)], np.uint64)
        if name in ("neg", "abs", "sqrt", "exp", "log", "sin", "cos", "floor"):
            dt = np.float64 if f else np.int64
            return np.asarray(O._BASE[name](xs[0].view(dt)), dt).view(np.uint64)
        if name == "select":
            return xs[1] if xs[0][0] != 0 else xs[2]
        if name == "dot":
            return _w(O._BASE["dot"](xs[0].view(np.float64)[None], xs[1].view(np.float64)[None])[0]).reshape(1)
        if name == "axpy":
            a = xs[0].view(np.float64)
            return (a[0] * xs[1].view(np.float64) + xs[2].view(np.float64)).view(np.uint64)
        if name in ("vget", "vstore"):
            k = int(as_i64(xs[1][0], vars_[ins[1]]["kind"]))
            w = len(xs[0])
            k = min(max(k, 0), w - 1)
            if name == "vget":
                return xs[0][k:k + 1]
            out = xs[0].copy()
            out[k] = xs[2][0]
            return out
        if name == "vcat":
            return np.concatenate(xs)
        if name == "vfill":
            return np.repeat(xs[0], int(op["width"]))
        if name == "vslice":
            lo = int(op["imm0"])
            return xs[0][lo:lo + int(op["width"])]
        if name == "rng_uniform":
            k = as_i64(xs[0][0], vars_[ins[0]]["kind"])
            c = as_i64(xs[1][0], vars_[ins[1]]["kind"])
            return O.rng_uniform(np.array([k]), np.array([c])).view(np.uint64)
        if name == "normals":  # fused draw_normals: the reference op sequence per pair
            key = as_i64(xs[0][0], vars_[ins[0]]["kind"])
            c = xs[1].view(np.float64)[0]
            k, pairs = int(op["imm0"]), int(op["imm1"])
            out = np.zeros(k + 1, np.float64)
            for pr in range(pairs):
                ua, ub = (O.rng_uniform(np.array([key]), np.array([as_i64(_w(c + float(j)), 0)]))[0]
                          for j in (2 * pr, 2 * pr + 1))
                r = np.sqrt(0.0 - 2.0 * np.log(1.0 - ua))
                out[2 * pr] = r * np.cos(6.283185307179586 * ub)
                if 2 * pr + 1 < k:
                    out[2 * pr + 1] = r * np.sin(6.283185307179586 * ub)
            out[k] = c + float(2 * pairs)
            return out.view(np.uint64)
        if name in ("logpdf", "grad"):
            t = targets[int(op["imm0"])]
            x = xs[0].view(np.float64)[None]
            if t.kind == 1:
                r = O.gaussian_logpdf(x, t.params["prec"], t.params["norm"]) if name == "logpdf" \
                    else O.gaussian_grad(x, t.params["prec"])
            else:
                r = O.logreg_logpdf(x, t.params["sx"]) if name == "logpdf" else O.logreg_grad(x, t.params["sx"])
            return np.asarray(r, np.float64).reshape(-1).view(np.uint64)
    raise NotImplementedError(name)


def run(dp, inputs: list[np.ndarray], depth: int):
    """All lanes; returns (outputs as uint64 words [z, w], per-lane block lists)."""
    z = inputs[0].shape[0]
    words = []
    for a in inputs:
        a = a.astype(np.uint64) if a.dtype == np.bool_ else a
        words.append(np.ascontiguousarray(a).view(np.uint64).reshape(z, -1))
    outs, traces = [], []
    for lane in range(z):
        o, tr = run_lane(dp, [w[lane] for w in words], depth)
        outs.append(o)
        traces.append(tr)
    return np.stack(outs), traces
