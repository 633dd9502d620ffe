"""CPU oracle: numpy restatement of the reference pc engine and its kernels.

TEST INFRASTRUCTURE ONLY. Nothing in `paper_1910_11141_b200/` imports this
module; only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU
baseline / `--impl reference` leg may use it, and only as the checker or the
timed CPU reference — never as the product path.

It re-states, in masked mode, the reference engine of arXiv 1910.11141's
`lockstep` package (`/root/reference/pkg/src/lockstep`):

* `step` — min-pc block selection, masked op execution by storage class,
  terminators, fault naming (`pc_vm.py:219-332`);
* `StackedVar` push / pop / write_top with a write-through cached top
  (`runtime.py:442-512`);
* every primitive kernel (`runtime.py:226-402`): numpy ufuncs, `dot` as
  `(a*b).sum(axis=1)`, `axpy` as `a[:, None]*x + y`, clipped `vget` /
  `vstore`, `rng_uniform` (`runtime.py:280-303`);
* target kernels (`workloads.py:186-228`): gaussian `norm - 0.5*einsum`,
  `-(x @ P)`; logistic `logaddexp` / stable sigmoid with two GEMMs.

It consumes the flat program of the reference's own compiler (the package
imports the installed `lockstep`, paper_1910_11141_b200/reference.py) and
re-states the engine and kernels independently of the reference's engine
code, so it can check the device on the GPU box.

Parity is pinned: `tests/test_oracle.py` checks this oracle bit-for-bit
against fixtures minted from the real reference (`tests/golden/make_golden.py`):
corpus outputs and step traces, NUTS chains, per-lane pc traces, rng
known-answer vectors, `dot` and einsum summation orders.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_U64 = np.uint64
_INV_2_53 = np.float64(1.0 / (1 << 53))


# ---- primitive kernels (reference runtime.py:226-402) ------------------------------------


def rng_uniform(key: np.ndarray, counter: np.ndarray) -> np.ndarray:
    """runtime.py:288-303."""
    k = key.astype(np.int64).astype(_U64)
    c = counter.astype(np.int64).astype(_U64)
    z = k * _U64(0xA24BAED4963EE407) + c * _U64(0x9E3779B97F4A7C15)
    z ^= z >> _U64(30)
    z *= _U64(0xBF58476D1CE4E5B9)
    z ^= z >> _U64(27)
    z *= _U64(0x94D049BB133111EB)
    z ^= z >> _U64(31)
    return (z >> _U64(11)).astype(np.float64) * _INV_2_53


def _clip_index(i, width):
    return np.clip(i.astype(np.int64), 0, width - 1)


def _div(a, b):
    if a.dtype == np.int64:
        return np.floor_divide(a, b)
    return np.divide(a, b)


def _select(c, a, b):
    return np.where(c if a.ndim == 1 else c[:, None], a, b)


def _vget(v, i):
    return np.take_along_axis(v, _clip_index(i, v.shape[1])[:, None], axis=1)[:, 0]


def _vstore(v, i, x):
    out = v.copy()
    np.put_along_axis(out, _clip_index(i, v.shape[1])[:, None], x[:, None], axis=1)
    return out


_BASE = {
    "add": np.add, "sub": np.subtract, "mul": np.multiply, "min": np.minimum,
    "max": np.maximum, "div": _div, "le": np.less_equal, "lt": np.less, "eq": np.equal,
    "and": np.logical_and, "or": np.logical_or, "not": np.logical_not, "neg": np.negative,
    "abs": np.abs, "sqrt": np.sqrt, "exp": np.exp, "log": np.log, "sin": np.sin, "cos": np.cos,
    "floor": np.floor, "select": _select,
    "dot": lambda a, b: (a * b).sum(axis=1),
    "axpy": lambda a, x, y: a[:, None] * x + y,
    "vget": _vget, "vstore": _vstore,
    "vcat": lambda a, b: np.concatenate((a, b), axis=1),
    "id": lambda a: a.copy(),
    "rng_uniform": rng_uniform,
}


def gaussian_logpdf(x, prec, norm):
    """workloads.py:188-189."""
    return norm - 0.5 * np.einsum("zi,ij,zj->z", x, prec, x)


def gaussian_grad(x, prec):
    """workloads.py:191-192."""
    return -(x @ prec)


def logreg_logpdf(w, sx):
    """workloads.py:216-219."""
    margins = w @ sx.T
    loglik = -np.logaddexp(0.0, -margins).sum(axis=1)
    return loglik - 0.5 * (w * w).sum(axis=1)


def logreg_grad(w, sx):
    """workloads.py:221-228."""
    margins = w @ sx.T
    with np.errstate(over="ignore"):
        sig = np.where(margins >= 0,
                       np.exp(-np.clip(margins, 0, None)) / (1.0 + np.exp(-np.clip(margins, 0, None))),
                       1.0 / (1.0 + np.exp(np.clip(margins, None, 0))))
    return sig @ sx - w


def kernel_for(name: str, targets: dict):
    """Resolve a primitive name to a numpy function over full-width batches."""
    if name in _BASE:
        return _BASE[name]
    head = name.split(":", 1)[0]
    if head == "const":
        _, kind, text = name.split(":", 2)
        val = {"i64": lambda: np.int64(int(text)), "f64": lambda: np.float64(float(text)),
               "bool": lambda: np.bool_(text == "true")}[kind]()
        return ("const", val)
    if head == "vfill":
        w = int(name.split(":")[1])
        return lambda a: np.repeat(a[:, None], w, axis=1)
    if head == "vslice":
        _, lo, hi = name.split(":")
        lo, hi = int(lo), int(hi)
        return lambda a: a[:, lo:hi].copy()
    for prefix in ("logpdf_", "grad_"):
        if name.startswith(prefix):
            t = targets[name[len(prefix):]]
            if t.kind == 1:
                prec, norm = t.params["prec"], t.params["norm"]
                return (lambda x: gaussian_logpdf(x, prec, norm)) if prefix == "logpdf_" else \
                    (lambda x: gaussian_grad(x, prec))
            sx = t.params["sx"]
            return (lambda w: logreg_logpdf(w, sx)) if prefix == "logpdf_" else (lambda w: logreg_grad(w, sx))
    raise KeyError(name)


# ---- stacks (reference runtime.py:442-512) -------------------------------------------------


class OracleFault(Exception):
    def __init__(self, kind: str, variable: str, lane: int, block: str | None = None):
        super().__init__(f"{kind} on '{variable}' lane {lane} in {block}")
        self.kind, self.variable, self.lane, self.block = kind, variable, lane, block


class StepLimit(Exception):
    pass


class Stack:
    def __init__(self, name, depth, z, dtype, lane_shape):
        self.name, self.depth = name, depth
        self.data = np.zeros((depth, z) + lane_shape, dtype=dtype)
        self.pointers = np.zeros(z, dtype=np.int64)
        self.cached_top = np.zeros((z,) + lane_shape, dtype=dtype)

    def push(self, values, mask):
        lanes = np.flatnonzero(mask)
        if lanes.size == 0:
            return
        ptrs = self.pointers[lanes]
        over = ptrs >= self.depth
        if over.any():
            raise OracleFault("overflow", self.name, int(lanes[over][0]))
        self.data[ptrs, lanes] = values[lanes]
        self.pointers[lanes] = ptrs + 1
        self.cached_top[lanes] = values[lanes]

    def pop(self, mask):
        lanes = np.flatnonzero(mask)
        if lanes.size == 0:
            return
        ptrs = self.pointers[lanes]
        under = ptrs < 1
        if under.any():
            raise OracleFault("underflow", self.name, int(lanes[under][0]))
        ptrs = ptrs - 1
        self.pointers[lanes] = ptrs
        live = ptrs >= 1
        if live.any():
            ll = lanes[live]
            self.cached_top[ll] = self.data[ptrs[live] - 1, ll]

    def write_top(self, values, mask):
        lanes = np.flatnonzero(mask)
        if lanes.size == 0:
            return
        ptrs = self.pointers[lanes]
        under = ptrs < 1
        if under.any():
            raise OracleFault("underflow", self.name, int(lanes[under][0]))
        self.data[ptrs - 1, lanes] = values[lanes]
        self.cached_top[lanes] = values[lanes]


# ---- the engine (reference pc_vm.py:140-383) ---------------------------------------------------


@dataclass
class OracleResult:
    output: np.ndarray
    steps: list            # (block index, active count) per step
    lane_blocks: list | None
    stack_ops: dict


def run(compiled, inputs, *, depth: int, types: dict, targets: dict, max_steps: int | None = 1_000_000,
        lane_traces: bool = False, observer=None, chooser=None) -> OracleResult:
    """Masked-mode pc engine: one min-pc block per step until every lane halts.

    `compiled` is a CompiledProgram (flat IR + classes + labels), `types` the
    inferred VType per variable, `targets` maps target name -> TargetDensity.
    `chooser(tops, depths) -> (block, selected mask)` replaces the min-pc rule
    (tests of the device's other schedules; per-lane results must not change).
    """
    flat, classes = compiled.flat, compiled.classes
    z = inputs[0].shape[0]
    halt = len(flat.blocks)

    def dtype_of(v):
        vt = types.get(v)
        return (np.float64, (vt.width,) if vt.width else ()) if vt is not None and vt.kind == "f64" \
            else ((np.bool_, ()) if vt is not None and vt.kind == "bool" else (np.int64, ()))

    stacks, plain = {}, {}
    for v, c in classes.items():
        dt, shape = dtype_of(v)
        if c == "stacked":
            s = Stack(v, depth, z, dt, shape)
            s.pointers[:] = 1
            stacks[v] = s
        else:
            plain[v] = np.zeros((z,) + shape, dtype=dt)
    for v, a in zip(flat.inputs, inputs):
        if v in stacks:
            stacks[v].data[0] = a
            stacks[v].cached_top[:] = a
        else:
            plain[v][:] = a
    pc = Stack("$pc", depth + 1, z, np.int64, ())
    pc.data[0] = halt
    pc.data[1] = flat.entry
    pc.pointers[:] = 2
    pc.cached_top[:] = flat.entry

    def value(v):
        return stacks[v].cached_top if v in stacks else plain[v]

    kernels = {}
    steps, stack_ops = [], {}
    lane_blocks = [[] for _ in range(z)] if lane_traces else None

    def note(var, kind):
        per = stack_ops.setdefault(var, {"push": 0, "pop": 0, "update": 0})
        per[kind] += 1

    from paper_1910_11141_b200 import ir  # IR node types only

    n = 0
    while True:
        tops = pc.cached_top
        active = tops != halt
        if not active.any():
            break
        if chooser is None:
            b = int(tops[active].min())
            sel = active & (tops == b)
        else:
            b, sel = chooser(tops, pc.pointers)
        steps.append((b, int(sel.sum())))
        if lane_blocks is not None:
            for lane in np.flatnonzero(sel):
                lane_blocks[lane].append(b)
        blk = flat.blocks[b]
        try:
            for op in blk.ops:
                if isinstance(op, ir.Pop):
                    note(op.var, "pop")
                    stacks[op.var].pop(sel)
                    continue
                k = kernels.get(op.prim.name)
                if k is None:
                    k = kernels[op.prim.name] = kernel_for(op.prim.name, targets)
                with np.errstate(all="ignore"):
                    if isinstance(k, tuple):
                        res = np.full(z, k[1], dtype=np.asarray(k[1]).dtype)
                    else:
                        res = k(*(value(v) for v in op.inputs))
                out = op.output
                if out in stacks:
                    if isinstance(op, ir.Push):
                        note(out, "push")
                        stacks[out].push(res, sel)
                    else:
                        note(out, "update")
                        stacks[out].write_top(res, sel)
                elif classes[out] == "register":
                    plain[out][sel] = res[sel]
                else:
                    plain[out][:] = res
            t = blk.terminator
            if isinstance(t, ir.FlatJump):
                pc.write_top(np.full(z, t.target, np.int64), sel)
            elif isinstance(t, ir.FlatBranch):
                pc.write_top(np.where(value(t.cond), t.true_target, t.false_target).astype(np.int64), sel)
            elif isinstance(t, ir.PushJump):
                pc.write_top(np.full(z, t.return_to, np.int64), sel)
                pc.push(np.full(z, t.jump_to, np.int64), sel)
            else:
                pc.pop(sel)
        except OracleFault as e:
            e.block = compiled.labels[b]
            raise
        n += 1
        if observer is not None:
            observer(b, sel, stacks, plain, pc)
        if max_steps is not None and n >= max_steps and (pc.cached_top != halt).any():
            raise StepLimit(max_steps)
    return OracleResult(value(flat.output).copy(), steps, lane_blocks, stack_ops)


# ---- the local-static engine (reference local_exec.py:81-185, Alg. 1) -----------------------


def run_local(program, inputs, *, targets: dict, max_steps: int | None = 1_000_000):
    """Masked-mode restatement of `run_local` on a CallGraphProgram.

    One activation of a function runs as a batched frame: every lane holds its
    own block cursor, each step runs the lowest populated block (min-pc
    chooser, local_exec.py:44-46) under the lane mask, and a call recurses on
    the host with the current mask (local_exec.py:81-128). Returns (output,
    steps) with one (label "fn.block", active lanes, grad invocations) per step.
    """
    from paper_1910_11141_b200 import ir  # IR node types only

    z = inputs[0].shape[0]
    grads = {t.grad for t in targets.values()}
    steps: list = []
    kernels: dict = {}

    def kernel(name):
        k = kernels.get(name)
        if k is None:
            k = kernels[name] = kernel_for(name, targets)
        return k

    def store(env, name, res, mask):
        dest = env.get(name)
        if dest is None:
            dest = env[name] = np.zeros_like(res)
        dest[mask] = res[mask]

    def call(fidx, args, live):
        fn = program.functions[fidx]
        halt = len(fn.blocks)
        env = {p: np.array(a, copy=True) for p, a in zip(fn.params, args)}
        pc = np.where(live, 0, halt).astype(np.int64)
        while True:
            cand = pc < halt
            if not cand.any():
                break
            b = int(pc[cand].min())
            sel = cand & (pc == b)
            if max_steps is not None and len(steps) >= max_steps:
                raise StepLimit(max_steps)
            block = fn.blocks[b]
            g = sum(1 for op in block.ops if isinstance(op, ir.Primitive) and op.prim.name in grads)
            steps.append((f"{fn.name}.{b}", int(sel.sum()), g))
            for op in block.ops:
                if isinstance(op, ir.Primitive):
                    k = kernel(op.prim.name)
                    with np.errstate(all="ignore"):
                        if isinstance(k, tuple):
                            res = np.full(z, k[1], dtype=np.asarray(k[1]).dtype)
                        else:
                            res = k(*(env[a] for a in op.inputs))
                    store(env, op.output, np.asarray(res), sel)
                else:
                    ret = call(op.callee, tuple(env[a] for a in op.args), sel)
                    store(env, op.output, ret, sel)
            t = block.terminator
            if isinstance(t, ir.Jump):
                pc[sel] = t.target
            elif isinstance(t, ir.Branch):
                pc[sel] = np.where(env[t.cond][sel], t.true_target, t.false_target)
            else:
                pc[sel] = halt
        out = env.get(fn.output)
        return np.zeros(z, dtype=np.int64) if out is None else out

    return call(program.entry, tuple(inputs), np.ones(z, dtype=bool)), steps


def utilization(steps, z: int) -> float:
    """metrics.utilization (reference metrics.py:52-76) over (label, active, grads) steps."""
    useful = sum(a * g for _, a, g in steps)
    launched = sum(z * g for _, _, g in steps)
    return useful / launched
