"""Drop-in replacement of the reference engine `lockstep.pc_vm`, on the B200.

Same entry points and semantics as reference `pkg/src/lockstep/pc_vm.py`:

    infer_types(flat, input_types)                           pc_vm.py:49-97 (the reference's own)
    init_machine(compiled, inputs, *, depth, mode, trace)    pc_vm.py:140-213
    step(m, *, observer, debug) -> bool                      pc_vm.py:304-332
    run_vm(m, *, max_steps, observer, debug)                 pc_vm.py:338-349
    run_flat(...), run(...) -> (outputs, ScheduleTrace)      pc_vm.py:352-383
    check_coherence(m)                                       pc_vm.py:391-400

Every block step executes in the CUDA VM (`csrc/engine.cu`) through the C ABI;
this module only moves inputs/outputs, maps status codes to the reference
exceptions and rebuilds `ScheduleTrace` records from the device trace.

Schedules. With Z <= 1024 lanes and no `lanes_per_group`, all lanes form one
schedule group and the device applies the reference's min-pc rule, so the
global step sequence (and every frozen step count) equals the reference's.
Larger batches are split into groups of `lanes_per_group` lanes (one CTA
each) that schedule independently and refill lanes from a chain queue; each
lane's results are unchanged (lane isolation, reference runtime.py:96-104),
and the returned trace carries per-block totals instead of a step list.

`mode` ("masked" / "gather") is accepted for API compatibility: the device
always computes only the selected lanes, which the reference guarantees to
be bit-identical to masked execution (test_acceptance.py:177-198).
"""

from __future__ import annotations

import numpy as np

from . import _native, ir
from . import schedule as _schedule
from .compiler import CompiledProgram
from .errors import StackFault, StackOverflow, StackUnderflow, StepLimitExceeded
from .lowering import DeviceProgram, lower
from .metrics import DeviceTrace, ScheduleTrace
from .reference import pc_vm as _ref_pc_vm
from .runtime import I64, VType, batch, vtype_of, words

DEFAULT_MAX_STEPS = 1_000_000
MAX_GROUP_LANES = 1024
# lowered programs (per compiled program and input types) and idle device machines
_PROGRAM_CACHE: dict = {}
_MACHINE_CACHE: dict = {}


# ---- type inference: the reference's own (pc_vm.py:49-97), used unchanged ---------------------

infer_types = _ref_pc_vm.infer_types


# ---- host views of device storage (for observers) -------------------------------------------


def _decode(raw: np.ndarray, vt: VType) -> np.ndarray:
    if vt.kind == "f64":
        arr = raw.view(np.float64)
    elif vt.kind == "i64":
        arr = raw.view(np.int64)
    else:
        arr = raw != 0
    return arr if vt.width else arr[..., 0]


class StackView:
    """Read-only snapshot of one stacked variable, shaped like runtime.StackedVar."""

    def __init__(self, name: str, depth: int, z: int, vt: VType, data: np.ndarray, pointers: np.ndarray):
        self.name, self.depth, self.z, self.vt = name, depth, z, vt
        self.data = data
        self.pointers = pointers

    @property
    def cached_top(self) -> np.ndarray:
        slot = np.maximum(self.pointers - 1, 0)
        return self.data[slot, np.arange(self.z)]


class _Views:
    def __init__(self, m: "Machine", cls: str):
        self.m, self.cls = m, cls

    def _names(self):
        return [v for v, c in self.m.classes.items() if c == self.cls]

    def __contains__(self, name):
        return self.m.classes.get(name) == self.cls

    def __iter__(self):
        return iter(self._names())

    def keys(self):
        return self._names()

    def values(self):
        return [self[n] for n in self._names()]

    def items(self):
        return [(n, self[n]) for n in self._names()]

    def __len__(self):
        return len(self._names())

    def __getitem__(self, name: str):
        if self.m.classes.get(name) != self.cls:
            raise KeyError(name)
        return self.m._view(name)


class GroupTrace(ScheduleTrace):
    """Trace of a multi-group run: per-block totals instead of one record per step.

    `block_steps[b]` counts group-steps of block b summed over groups,
    `block_active[b]` the active lanes they carried; `lanes` is the group width.
    """

    def __init__(self, engine: str, z: int, labels, prims, lanes: int,
                 block_steps: np.ndarray, block_active: np.ndarray):
        super().__init__(engine=engine, z=z)
        self.labels, self.block_prims, self.lanes = labels, prims, lanes
        self.block_steps, self.block_active = block_steps, block_active

    @property
    def step_count(self) -> int:
        return int(self.block_steps.sum())

    device_grads: np.ndarray | None = None  # per-block grads of the program the device ran
    grad_names: frozenset = frozenset()

    def _per_block(self, counted):
        if counted and self.device_grads is not None and set(counted) <= self.grad_names:
            # fused superblocks move a function's gradients into its entry block
            return self.device_grads.astype(np.int64)
        return np.array([sum(n for k, n in p.items() if counted is None or k in counted)
                         for p in self.block_prims], dtype=np.int64)

    def invocations(self, counted=None) -> int:
        return int((self.block_steps * self._per_block(counted)).sum())

    def useful_invocations(self, counted=None) -> int:
        return int((self.block_active * self._per_block(counted)).sum())

    def occupancy(self, counted=None) -> tuple[int, int]:
        c = self._per_block(counted)
        return int((self.block_active * c).sum()), int((self.block_steps * c).sum()) * self.lanes


# ---- the machine ----------------------------------------------------------------------------


class Machine:
    """A batch of Z lanes resident on the GPU (reference `Machine`, pc_vm.py:103-137)."""

    def __init__(self, compiled: CompiledProgram, dp: DeviceProgram, handle: _native.MachineHandle,
                 z: int, depth: int, mode: str, types, trace: ScheduleTrace | None,
                 schedule: str, groups_exact: bool, lanes: int):
        self.flat = compiled.flat
        self.classes = dp.classes
        self.labels = compiled.labels
        self.z, self.depth, self.mode, self.types = z, depth, mode, types
        self.trace = trace
        self.steps = 0
        self.schedule = schedule
        self.exact = groups_exact
        self.lanes = lanes
        self._dp = dp
        self._h = handle
        self._useful = 0
        self._launched = 0
        self.stacks = _Views(self, "stacked")
        self.regs = _Views(self, "register")
        self.scratch = _Views(self, "temporary")
        self.halted = False
        self.engine = "exact"

    @property
    def halt_index(self) -> int:
        return self.flat.halt_index

    def lane_traces(self) -> list[np.ndarray]:
        """Each lane's executed block sequence (needs lane_trace_cap > 0 at init)."""
        return self._h.lane_traces()

    def group_traces(self) -> list[ScheduleTrace]:
        """Warp engine (group_trace_cap > 0 at init): one reference ScheduleTrace per
        32-lane group — StepRecord(block label, active lanes, prims) per step and the
        per-variable stack-op counts (reference metrics.py:29-41), so utilization(),
        compare() and trace_to_json() apply per group. Fused superblocks carry their
        function's gradient count; a paired step appears as two records."""
        from .lowering import grad_names

        dp = self._dp
        gnames = grad_names()
        prims = []
        for b, p in enumerate(dp.block_prims):
            p = {k: v for k, v in p.items() if k not in gnames}
            g = int(dp.blocks["grads"][b])
            if g:  # the device's count (a fused superblock does its function's gradients)
                fn = self.labels[b].split(".", 1)[0]
                names = [k for k in dp.block_prims[b] if k in gnames] or \
                        [k for c, q in enumerate(dp.block_prims) if self.labels[c].split(".", 1)[0] == fn
                         for k in q if k in gnames]
                if names:
                    p[names[0]] = g
            prims.append(p)
        out = []
        width = min(32, self.z)  # a group's lanes (a batch of <= 32 chains is one group)
        for recs in self._h.group_traces():
            tr = ScheduleTrace(engine="pc", z=width)
            for r in recs:
                b, act = int(r) & 0xffff, int(r) >> 16
                tr.record(self.labels[b], act, prims[b])
                for var, kind in dp.block_stack_ops[b]:
                    tr.record_stack_op(var, kind)
            out.append(tr)
        return out

    @property
    def useful_grads(self) -> int:
        """Sum over steps of active lanes x grad invocations (the headline unit)."""
        return self._useful

    def _need_exact(self):
        if not self.exact:
            raise ValueError("machine state views need a single schedule group (Z <= 1024)")

    def _view(self, name: str):
        self._need_exact()
        vid = self._dp.var_index[name]
        vt = self._dp.types[name]
        cls = self.classes[name]
        slots = self.depth if cls == "stacked" else 1
        raw = self._h.read_var(vid, slots, words(vt))
        data = _decode(raw, vt)
        if cls == "stacked":
            return StackView(name, self.depth, self.z, vt, data, self._h.read_pointers(vid))
        return data[0]

    @property
    def pc(self) -> StackView:
        self._need_exact()
        data = self._h.read_pc_stack()
        return StackView("$pc", self.depth + 1, self.z, I64, data, self._h.read_pointers(-1))

    def value_of(self, var: str) -> np.ndarray:
        v = self._view(var)
        return v.cached_top if isinstance(v, StackView) else v

    def pc_tops(self) -> np.ndarray:
        return self.pc.cached_top

    def active_mask(self) -> np.ndarray:
        if self.exact:
            return self.pc_tops() != self.halt_index
        return np.zeros(self.z, bool) if self.halted else np.ones(self.z, bool)

    def output_value(self) -> np.ndarray:
        if self.halted or not self.exact:
            vt = self._dp.types[self.flat.output]
            # read_output hands back a fresh array (never aliased by the machine)
            return _decode(self._h.read_output(words(vt), np.uint64).reshape(self.z, words(vt)), vt)
        return np.array(self.value_of(self.flat.output), copy=True)


def _prepare_inputs(flat: ir.FlatProgram, inputs) -> list[np.ndarray]:
    arrays = [a if isinstance(a, np.ndarray) else batch(a) for a in inputs]
    if len(arrays) != len(flat.inputs):
        raise ValueError(f"program wants {len(flat.inputs)} inputs, got {len(arrays)}")
    if not arrays:
        raise ValueError("program must take at least one input")
    z = arrays[0].shape[0]
    if any(a.shape[0] != z for a in arrays):
        raise ValueError("all inputs must share the batch width")
    if z < 1:
        raise ValueError("batch width must be at least 1")
    return arrays


def _as_words(a: np.ndarray) -> np.ndarray:
    if a.dtype == np.bool_:
        a = a.astype(np.uint64)
    a = np.ascontiguousarray(a)
    return a.view(np.uint64).reshape(a.shape[0], -1)


ENGINES = ("auto", "exact", "cta", "warp")


def _pick_engine(engine: str, z: int, lanes_per_group: int | None) -> str:
    if engine not in ENGINES:
        raise ValueError(f"unknown engine '{engine}' (one of {ENGINES})")
    if engine != "auto":
        return engine
    if lanes_per_group is not None:
        return "cta"
    return "exact" if z <= MAX_GROUP_LANES else "warp"


def init_machine(compiled: CompiledProgram, inputs, *, depth: int, mode: str = "masked",
                 trace: ScheduleTrace | None = None, schedule: str = "min_pc",
                 lanes_per_group: int | None = None, groups: int = 0,
                 optimize: bool = False, exact_logpdf: bool = True,
                 lane_trace_cap: int = 0, engine: str = "auto",
                 codegen: bool | str = False, reuse: bool = False, device: int | None = None,
                 precision: str = "fp64", group_trace_cap: int = 0) -> Machine:
    """Allocate device storage and seed the batch (reference pc_vm.py:140-213).

    Data stacks get `depth` slots with one live slot per lane; inputs land in
    that slot; the pc stack gets depth+1 slots seeded [halt, entry].

    engine: "exact" — all Z (<= 1024) lanes in one CTA group, reference min-pc
    schedule, per-step trace, observers; "cta" — groups of `lanes_per_group`
    lanes, one CTA each; "warp" — the throughput engine: one 32-lane group per
    warp, DMMA target contractions, fused leapfrog superblocks (with
    optimize); "auto" picks exact for Z <= 1024, else warp.

    codegen (warp engine): run program-specialised block code (codegen.py)
    instead of the op interpreter; compiled once per program and cached
    in-tree ("cached": use only a prebuilt library).

    precision (warp engine): "fp64" — the reference's arithmetic (DMMA superblocks);
    "fp32" — fused leapfrogs in float32 on the tensor cores (tcgen05 kind::tf32, 3xTF32
    split; gaussian targets with d <= 128, 1e-5 relative per leapfrog step).
    device: CUDA device index the machine lives on (one process per GPU passes
    its LOCAL_RANK; None = the library's current device, 0 by default).
    schedule: block-selection rule (schedule.SCHEDULES): "min_pc" (reference),
    "most_populated", "local" (paper Alg. 1) or "priority" (throughput).
    group_trace_cap (warp engine): record each 32-lane group's first steps as the
    reference's per-step schedule trace (Machine.group_traces).
    """
    if mode not in ("masked", "gather"):
        raise ValueError(f"unknown mode '{mode}'")
    if depth < 1:
        raise ValueError("stack depth must be at least 1")
    from .compiler import adopt

    compiled = adopt(compiled)  # the reference compiler's CompiledProgram
    flat = compiled.flat
    arrays = _prepare_inputs(flat, inputs)
    z = arrays[0].shape[0]
    in_types = [vtype_of(a) for a in arrays]
    kind = _pick_engine(engine, z, lanes_per_group)
    if kind == "exact" and z > MAX_GROUP_LANES:
        raise ValueError(f"the exact engine holds at most {MAX_GROUP_LANES} lanes")
    pkey = (id(compiled), tuple(map(str, in_types)), optimize, kind == "warp",
            codegen if kind == "warp" else False, device)
    hit = _PROGRAM_CACHE.get(pkey)
    if hit is not None and hit[0] is compiled:
        dp, program, types = hit[1], hit[2], hit[3]
    else:
        types = infer_types(flat, in_types)
        dp = lower(compiled, types, optimize=optimize, superblocks=(kind == "warp"))
        lib = None
        if codegen and kind == "warp":
            from . import codegen as _cg

            lib = _cg.library_for(dp, build=codegen != "cached")
            if lib is None:
                raise ValueError("no prebuilt specialised library for this program (codegen='cached')")
        program = _native.Program(dp, lib, device=device)
        if len(_PROGRAM_CACHE) >= 16:
            _PROGRAM_CACHE.pop(next(iter(_PROGRAM_CACHE)))
        _PROGRAM_CACHE[pkey] = (compiled, dp, program, types)
    exact = kind == "exact"
    if kind == "cta" and lanes_per_group is None:
        lanes_per_group = 256
    lanes = z if exact else (32 if kind == "warp" else int(lanes_per_group))
    mopts = dict(sched=schedule, lanes_per_cta=int(lanes_per_group) if kind == "cta" else 0,
                 ctas=groups, trace=exact and trace is not None, exact_logpdf=exact_logpdf,
                 lane_trace_cap=lane_trace_cap, warp_groups=(kind == "warp"), precision=precision,
                 group_trace_cap=group_trace_cap)
    mkey = (pkey, z, depth, tuple(sorted(mopts.items())))
    handle = _MACHINE_CACHE.pop(mkey, None) if reuse else None
    if handle is not None and handle.program is program:
        handle.reset()
    else:
        handle = _native.MachineHandle(program, z, depth, **mopts)
    if reuse:  # run() hands the machine back to the cache when it is done with it
        handle.cache_key = mkey
    keys = _schedule.block_keys(flat, compiled.labels, schedule,
                                np.flatnonzero(np.asarray(dp.blocks["grads"]) > 0))
    handle.set_block_keys(keys)
    for k, a in enumerate(arrays):
        handle.set_input(k, _as_words(a))
    m = Machine(compiled, dp, handle, z, depth, mode, types, trace, schedule, exact, lanes)
    m.engine = kind
    m._keys = keys
    if not exact and trace is not None:
        m.trace = GroupTrace("pc", z, compiled.labels, dp.block_prims, lanes,
                             np.zeros(len(flat.blocks), np.int64), np.zeros(len(flat.blocks), np.int64))
        from .lowering import grad_names

        m.trace.device_grads = np.array(dp.blocks["grads"])
        m.trace.grad_names = grad_names()
    return m


def _raise_fault(m: Machine, st) -> None:
    label = m.labels[st.block] if 0 <= st.block < len(m.labels) else None
    if st.var < 0:
        name, cap = "$pc", m.depth + 1
    else:
        name, cap = m._dp.var_names[st.var], m.depth
    if st.kind == _native.RUN_OVERFLOW:
        err: StackFault = StackOverflow(name, int(st.lane), f"depth {cap}")
    else:
        err = StackUnderflow(name, int(st.lane), "update on empty stack" if st.pad == 1 else "")
    err.block = label
    raise err


def _record(m: Machine, blocks: np.ndarray, active: np.ndarray) -> None:
    tr = m.trace
    if tr is None or isinstance(tr, GroupTrace):
        return
    labels, prims, sops = m.labels, m._dp.block_prims, m._dp.block_stack_ops
    for b, n in zip(blocks.tolist(), active.tolist()):
        tr.record(labels[b], n, prims[b])
        for var, kind in sops[b]:
            tr.record_stack_op(var, kind)


def _absorb(m: Machine, st) -> None:
    m.steps = int(st.steps)
    m._useful = int(st.useful_grads)
    m._launched = int(st.launched_grads)
    if m.exact and m.trace is not None:
        b, a = m._h.fetch_trace()
        _record(m, b, a)


def step(m: Machine, *, observer=None, debug: bool = False) -> bool:
    """Execute one batched block on the device; False once every lane has halted."""
    m._need_exact()
    pc = m.pc
    tops = pc.cached_top
    active = tops != m.halt_index
    if not active.any():
        m.halted = True
        return False
    b, sel = _schedule.select(m.schedule, tops, pc.pointers, m._keys, m.halt_index)
    st = m._h.run(m.steps + 1)
    if st.kind in (_native.RUN_OVERFLOW, _native.RUN_UNDERFLOW):
        _absorb(m, st)
        _raise_fault(m, st)
    _absorb(m, st)
    if observer is not None:
        observer(m, b, sel)
    if debug:
        check_coherence(m)
        new = m.pc_tops()
        if (new[~active] != m.halt_index).any():
            raise AssertionError("halted lane resumed execution")
        if ((new < 0) | (new > m.halt_index)).any():
            raise AssertionError("pc top left the block range")
    return True


def run_vm(m: Machine, *, max_steps: int | None = DEFAULT_MAX_STEPS, observer=None,
           debug: bool = False) -> np.ndarray:
    """Step until every lane halts; returns the output batch (reference pc_vm.py:338-349)."""
    if observer is not None or debug:
        while step(m, observer=observer, debug=debug):
            if max_steps is not None and m.steps >= max_steps and m.active_mask().any():
                raise StepLimitExceeded(max_steps)
        return m.output_value()
    limit = -1 if max_steps is None else int(max_steps)
    while True:
        st = m._h.run(limit)
        _absorb(m, st)
        if st.kind == _native.RUN_HALTED:
            break
        if st.kind in (_native.RUN_OVERFLOW, _native.RUN_UNDERFLOW):
            _raise_fault(m, st)
        if st.kind == _native.RUN_STEP_LIMIT:
            raise StepLimitExceeded(max_steps)
        # RUN_PAUSED: trace buffer drained by _absorb; continue
    m.halted = True
    if isinstance(m.trace, GroupTrace):
        m.trace.block_steps, m.trace.block_active = m._h.block_totals(len(m.flat.blocks))
    return m.output_value()


def run_flat(compiled: CompiledProgram, inputs, *, depth: int, mode: str = "masked",
             max_steps: int | None = DEFAULT_MAX_STEPS, trace: ScheduleTrace | None = None,
             observer=None, debug: bool = False, **engine) -> np.ndarray:
    """init_machine + run_vm."""
    engine.setdefault("optimize", observer is None and not debug)
    m = init_machine(compiled, inputs, depth=depth, mode=mode, trace=trace, **engine)
    return run_vm(m, max_steps=max_steps, observer=observer, debug=debug)


def run(compiled: CompiledProgram, inputs, *, depth: int, mode: str = "masked",
        max_steps: int | None = DEFAULT_MAX_STEPS, observer=None, debug: bool = False,
        schedule: str = "min_pc", lanes_per_group: int | None = None, groups: int = 0,
        optimize: bool | None = None, exact_logpdf: bool = True, lane_trace_cap: int = 0,
        engine: str = "auto", codegen: bool | str = False, return_machine: bool = False,
        device: int | None = None, precision: str = "fp64", group_trace_cap: int = 0):
    """Execute a compiled program on the B200; returns (outputs, trace)."""
    arrays = [a if isinstance(a, np.ndarray) else batch(a) for a in inputs]
    z = arrays[0].shape[0] if arrays else 0
    if optimize is None:
        optimize = observer is None and not debug
    tr: ScheduleTrace = DeviceTrace(engine="pc", z=z)
    # device storage is reused across calls with the same program and shapes; a
    # machine handed back to the caller (return_machine) is not recycled
    reuse = not return_machine and observer is None and not debug
    m = init_machine(compiled, arrays, depth=depth, mode=mode, trace=tr, schedule=schedule,
                     lanes_per_group=lanes_per_group, groups=groups, optimize=optimize,
                     exact_logpdf=exact_logpdf, lane_trace_cap=lane_trace_cap, engine=engine,
                     codegen=codegen, reuse=reuse, device=device, precision=precision,
                     group_trace_cap=group_trace_cap)
    if m.engine == "warp" and observer is None and not debug and not return_machine:
        # output rows go straight to a pinned host buffer while the run executes (not for
        # a machine handed back: its device output must stay valid for later reads)
        m._h.stream_output_to_host(words(m._dp.types[m.flat.output]))
    try:
        out = run_vm(m, max_steps=max_steps, observer=observer, debug=debug)
    finally:
        if m._h._host_out is not None:  # a fault left the buffer unclaimed
            m._h._host_out = None
            m._h._c(m._h.lib.ls_machine_set_output_host(m._h.handle, None, 0))
        if reuse:
            if len(_MACHINE_CACHE) >= 4:
                _MACHINE_CACHE.pop(next(iter(_MACHINE_CACHE)))
            _MACHINE_CACHE[m._h.cache_key] = m._h
    if return_machine:
        return out, m.trace, m
    return out, m.trace


def trace_flat(compiled: CompiledProgram, inputs, *, depth: int, **kwargs):
    return run(compiled, inputs, depth=depth, **kwargs)


def check_coherence(m: Machine) -> None:
    """Debug invariant of the reference (pc_vm.py:391-400).

    The device keeps no separate cached top (the top is read from the slot
    under the pointer), so coherence reduces to pointers staying in range.
    """
    for name in list(m.stacks):
        sv = m.stacks[name]
        if ((sv.pointers < 0) | (sv.pointers > sv.depth)).any():
            raise AssertionError(f"stack pointer out of range on '{name}'")
    pc = m.pc
    if ((pc.pointers < 0) | (pc.pointers > pc.depth)).any():
        raise AssertionError("pc stack pointer out of range")
