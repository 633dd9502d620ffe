"""ctypes binding of `include/lockstep_b200.h` (the C ABI of the B200 VM).

This is the only place Python touches the CUDA library. It loads the
in-tree `_lib/liblockstep_b200.so` (or a program-specialised build of the
same ABI from `_lib/gen/`, see codegen.py) and fails loudly (DeviceError)
if the library or a GPU is missing: there is no CPU fallback behind it.
"""

from __future__ import annotations

import ctypes as C
import re
import sys
from pathlib import Path

import numpy as np

from .errors import DeviceError
from .lowering import DeviceProgram

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "liblockstep_b200.so"
HEADER = Path(__file__).resolve().parent.parent / "include" / "lockstep_b200.h"

LS_OK, LS_EINVAL, LS_ECUDA, LS_ENOMEM = 0, -1, -2, -3
RUN_HALTED, RUN_PAUSED, RUN_OVERFLOW, RUN_UNDERFLOW, RUN_STEP_LIMIT = 0, 1, 2, 3, 4
SCHED = {"min_pc": 0, "most_populated": 1, "local": 2, "priority": 3}
MF_NO_STAGE, MF_FP32 = 1, 2  # ls_machine_opts.flags (lockstep_b200.h)
PRECISIONS = ("fp64", "fp32")


class ProgramDesc(C.Structure):
    _fields_ = [("blocks", C.c_void_p), ("n_blocks", C.c_int32),
                ("ops", C.c_void_p), ("n_ops", C.c_int32),
                ("vars", C.c_void_p), ("n_vars", C.c_int32),
                ("entry", C.c_int32),
                ("inputs", C.c_void_p), ("n_inputs", C.c_int32),
                ("output", C.c_int32), ("flat_rows", C.c_int32)]


class MachineOpts(C.Structure):
    _fields_ = [("sched", C.c_int32), ("lanes_per_cta", C.c_int32), ("ctas", C.c_int32),
                ("trace", C.c_int32), ("exact_logpdf", C.c_int32), ("lane_trace_cap", C.c_int32),
                ("warp_groups", C.c_int32), ("flags", C.c_int32), ("group_trace_cap", C.c_int32)]


class Status(C.Structure):
    _fields_ = [("kind", C.c_int32), ("var", C.c_int32), ("lane", C.c_int64),
                ("block", C.c_int32), ("pad", C.c_int32), ("steps", C.c_int64),
                ("useful_grads", C.c_int64), ("launched_grads", C.c_int64),
                ("kernel_ms", C.c_double), ("launches", C.c_int64)]


_SIGS = {
    "ls_abi_version": ([], C.c_int),
    "ls_host_alloc": ([C.c_int64, C.POINTER(C.c_void_p)], C.c_int),
    "ls_host_free": ([C.c_void_p], C.c_int),
    "ls_machine_set_output_host": ([C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "ls_last_error": ([], C.c_char_p),
    "ls_device_count": ([C.POINTER(C.c_int32)], C.c_int),
    "ls_set_device": ([C.c_int32], C.c_int),
    "ls_machine_info": ([C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)], C.c_int),
    "ls_program_create": ([C.POINTER(ProgramDesc), C.POINTER(C.c_void_p)], C.c_int),
    "ls_program_bind_target": ([C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                C.c_void_p, C.c_double], C.c_int),
    "ls_program_destroy": ([C.c_void_p], C.c_int),
    "ls_machine_create": ([C.c_void_p, C.c_int64, C.c_int32, C.POINTER(MachineOpts),
                           C.POINTER(C.c_void_p)], C.c_int),
    "ls_machine_set_input": ([C.c_void_p, C.c_int32, C.c_void_p, C.c_int64], C.c_int),
    "ls_machine_reset": ([C.c_void_p], C.c_int),
    "ls_machine_set_block_keys": ([C.c_void_p, C.c_void_p, C.c_int32], C.c_int),
    "ls_machine_set_input_device": ([C.c_void_p, C.c_int32, C.c_void_p, C.c_int64], C.c_int),
    "ls_run": ([C.c_void_p, C.c_int64, C.POINTER(Status)], C.c_int),
    "ls_read_output": ([C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "ls_output_device": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "ls_copy_output_device": ([C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "ls_trace_fetch": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
    "ls_block_totals": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ls_block_cycles": ([C.c_void_p, C.c_void_p], C.c_int),
    "ls_read_var": ([C.c_void_p, C.c_int32, C.c_void_p, C.c_int64], C.c_int),
    "ls_read_pointers": ([C.c_void_p, C.c_int32, C.c_void_p, C.c_int64], C.c_int),
    "ls_read_pc_stack": ([C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "ls_lane_trace_fetch": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "ls_group_trace_fetch": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "ls_machine_sync": ([C.c_void_p], C.c_int),
    "ls_machine_destroy": ([C.c_void_p], C.c_int),
    "ls_rng_uniform": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p], C.c_int),
    "ls_target_eval": ([C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_double,
                        C.c_void_p, C.c_int64, C.c_void_p], C.c_int),
}

_LIBS: dict[str, C.CDLL] = {}


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(ls_\w+)\(", text, re.M)))


def load(path: Path | str | None = None) -> C.CDLL:
    """Load (never build) a CUDA library of this ABI; DeviceError if it is absent."""
    path = str(path or LIB_PATH)
    lib = _LIBS.get(path)
    if lib is not None:
        return lib
    if not Path(path).exists():
        raise DeviceError(f"CUDA library {path} is missing; run "
                          "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _LIBS[path] = lib
    return lib


def _check(rc: int, lib: C.CDLL | None = None) -> None:
    if rc != LS_OK:
        msg = (lib or load()).ls_last_error().decode(errors="replace")
        if rc == LS_EINVAL:
            raise ValueError(msg)
        raise DeviceError(msg)


def device_count() -> int:
    n = C.c_int32(0)
    rc = load().ls_device_count(C.byref(n))
    return n.value if rc == LS_OK else 0


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class Program:
    """Owns an `ls_program` built from a DeviceProgram (in library `lib_path`)."""

    def __init__(self, dp: DeviceProgram, lib_path: Path | str | None = None, device: int | None = None):
        self.lib = load(lib_path)
        self.lib_path = str(lib_path or LIB_PATH)
        self.dp = dp
        if device is not None:  # the program (and its machines) live on this CUDA device
            _check(self.lib.ls_set_device(int(device)), self.lib)
        self.device = device
        self._keep = [np.ascontiguousarray(dp.blocks), np.ascontiguousarray(dp.ops),
                      np.ascontiguousarray(dp.vars), np.ascontiguousarray(dp.inputs, dtype=np.int32)]
        b, o, v, i = self._keep
        desc = ProgramDesc(_ptr(b), len(b), _ptr(o) if len(o) else None, len(o), _ptr(v), len(v),
                           dp.flat.entry, _ptr(i) if len(i) else None, len(i), dp.output,
                           dp.flat_rows)
        h = C.c_void_p()
        _check(self.lib.ls_program_create(C.byref(desc), C.byref(h)), self.lib)
        self.handle = h
        for slot, t in enumerate(dp.targets):
            self._bind(slot, t)

    def _bind(self, slot: int, t) -> None:
        from .workloads import TARGET_GAUSSIAN

        if t.kind == TARGET_GAUSSIAN:
            params, n, norm = t.params["prec"], t.dim, t.params["norm"]
        else:
            params, n, norm = t.params["sx"], t.params["sx"].shape[0], 0.0
        params = np.ascontiguousarray(params, dtype=np.float64)
        _check(self.lib.ls_program_bind_target(self.handle, slot, t.kind, t.dim, n, _ptr(params), norm),
               self.lib)

    def __del__(self):
        if getattr(self, "handle", None):
            self.lib.ls_program_destroy(self.handle)
            self.handle = None


class _PinnedBuf:
    """One page-locked host allocation (ls_host_alloc); freed when unreferenced."""

    __slots__ = ("lib", "ptr", "nbytes")

    def __init__(self, lib, nbytes: int):
        p = C.c_void_p()
        _check(lib.ls_host_alloc(nbytes, C.byref(p)), lib)
        self.lib, self.ptr, self.nbytes = lib, p.value, nbytes

    def __del__(self):
        try:
            self.lib.ls_host_free(C.c_void_p(self.ptr))
        except Exception:  # interpreter teardown
            pass


class _HostView:
    """numpy base object that keeps a pinned buffer alive while any view exists."""

    def __init__(self, buf: _PinnedBuf, shape: tuple[int, ...]):
        self.buf = buf
        self.__array_interface__ = {"data": (buf.ptr, False), "shape": shape, "typestr": "<u8",
                                    "version": 3}


class HostPool:
    """Page-locked destinations for large output reads (a caching host allocator).

    ls_read_output into pinned memory is one DMA at PCIe rate, while a fresh
    pageable array costs first-touch page faults plus the driver's staging copy.
    A buffer is handed out again only when no array returned from it is still
    referenced (its refcount is back to the pool's own), so results a caller
    keeps are never overwritten; when every buffer is busy the pool grows up to
    `cap` buffers per size, then callers fall back to ordinary numpy memory.
    """

    def __init__(self, cap: int = 3, min_bytes: int = 1 << 22):
        self.cap, self.min_bytes = cap, min_bytes
        self.bufs: dict[int, list[_PinnedBuf]] = {}

    def array(self, lib, shape: tuple[int, ...]) -> np.ndarray | None:
        nbytes = int(np.prod(shape)) * 8
        if nbytes < self.min_bytes:
            return None
        free = self.bufs.setdefault(nbytes, [])
        for b in free:
            if sys.getrefcount(b) <= 3:  # the list, the loop variable, the call argument
                return np.asarray(_HostView(b, shape))
        if len(free) >= self.cap:
            return None
        try:
            b = _PinnedBuf(lib, nbytes)
        except DeviceError:
            return None
        free.append(b)
        return np.asarray(_HostView(b, shape))


HOST_POOL = HostPool()


class MachineHandle:
    """Owns an `ls_machine` (device storage for one batch of lanes)."""

    def __init__(self, program: Program, z: int, depth: int, *, sched: str = "min_pc",
                 lanes_per_cta: int = 0, ctas: int = 0, trace: bool = False,
                 exact_logpdf: bool = True, lane_trace_cap: int = 0, warp_groups: bool = False,
                 stage_targets: bool = True, precision: str = "fp64", group_trace_cap: int = 0):
        if sched not in SCHED:
            raise ValueError(f"unknown schedule '{sched}'")
        self.program = program
        self.lib = program.lib
        self.z = z
        self.depth = depth
        opts = MachineOpts(SCHED[sched], lanes_per_cta, ctas, int(trace), int(exact_logpdf),
                           int(lane_trace_cap), int(warp_groups),
                           (0 if stage_targets else MF_NO_STAGE) | (MF_FP32 if precision == "fp32" else 0),
                           int(group_trace_cap))
        if precision not in PRECISIONS:
            raise ValueError(f"unknown precision '{precision}' (one of {PRECISIONS})")
        if precision == "fp32" and not warp_groups:
            raise ValueError("the fp32 arm runs on the warp engine (engine='warp')")
        self.precision = precision
        self.lane_trace_cap = int(lane_trace_cap)
        self.group_trace_cap = int(group_trace_cap)
        self.warp_groups = bool(warp_groups)
        self._host_out: np.ndarray | None = None
        h = C.c_void_p()
        _check(self.lib.ls_machine_create(program.handle, z, depth, C.byref(opts), C.byref(h)), self.lib)
        self.handle = h

    def _c(self, rc):
        _check(rc, self.lib)

    def set_input(self, idx: int, arr: np.ndarray) -> None:
        arr = np.ascontiguousarray(arr)
        self._c(self.lib.ls_machine_set_input(self.handle, idx, _ptr(arr), arr.nbytes))

    def reset(self) -> None:
        self._c(self.lib.ls_machine_reset(self.handle))

    def info(self) -> tuple[int, int, int]:
        """(CUDA device, schedule groups, lanes per group)."""
        d, g, l = C.c_int32(), C.c_int32(), C.c_int32()
        self._c(self.lib.ls_machine_info(self.handle, C.byref(d), C.byref(g), C.byref(l)))
        return d.value, g.value, l.value

    @property
    def groups(self) -> int:
        return self.info()[1]

    @property
    def device(self) -> int:
        return self.info()[0]

    def set_block_keys(self, keys: np.ndarray) -> None:
        keys = np.ascontiguousarray(keys, dtype=np.uint32)
        self._c(self.lib.ls_machine_set_block_keys(self.handle, _ptr(keys), len(keys)))

    def set_input_device(self, idx: int, dev_ptr: int, nbytes: int) -> None:
        self._c(self.lib.ls_machine_set_input_device(self.handle, idx, C.c_void_p(dev_ptr), nbytes))

    def run(self, max_steps: int) -> Status:
        st = Status()
        self._c(self.lib.ls_run(self.handle, max_steps, C.byref(st)))
        return st

    def stream_output_to_host(self, width: int) -> bool:
        """Warp engine: let the next run write its output rows straight into a pinned
        pool buffer (the PCIe transfer overlaps the run). False if none is free."""
        if not self.warp_groups:
            return False
        out = HOST_POOL.array(self.lib, (self.z, width))
        if out is None:
            return False
        self._c(self.lib.ls_machine_set_output_host(self.handle, _ptr(out), out.nbytes))
        self._host_out = out
        return True

    def read_output(self, width: int, dtype) -> np.ndarray:
        """A fresh host array of the output (pinned from HOST_POOL when large)."""
        if self._host_out is not None:  # already in host memory: synchronise, hand it over
            out, self._host_out = self._host_out, None
            try:
                self._c(self.lib.ls_read_output(self.handle, _ptr(out), out.nbytes))
            finally:
                self._c(self.lib.ls_machine_set_output_host(self.handle, None, 0))
            return out.view(dtype)
        out = HOST_POOL.array(self.lib, (self.z, width))
        if out is None:
            out = np.empty((self.z, width), dtype=np.uint64)
        self._c(self.lib.ls_read_output(self.handle, _ptr(out), out.nbytes))
        return out.view(dtype)

    def copy_output_rows_to(self, dev_ptr: int, rows: int) -> None:
        """The first `rows` output rows into device memory at dev_ptr."""
        width = int(self.program.dp.vars[self.program.dp.output]["width"])
        self._c(self.lib.ls_copy_output_device(self.handle, C.c_void_p(dev_ptr), rows * width * 8))

    def copy_output_to(self, dev_ptr: int, nbytes: int) -> None:
        self._c(self.lib.ls_copy_output_device(self.handle, C.c_void_p(dev_ptr), nbytes))

    def output_device_ptr(self) -> int:
        p = C.c_void_p()
        self._c(self.lib.ls_output_device(self.handle, C.byref(p)))
        return p.value

    def fetch_trace(self, cap: int = 1 << 16) -> tuple[np.ndarray, np.ndarray]:
        blocks, active = [], []
        while True:
            b = np.empty(cap, np.int32)
            a = np.empty(cap, np.int32)
            n = C.c_int64(0)
            self._c(self.lib.ls_trace_fetch(self.handle, _ptr(b), _ptr(a), cap, C.byref(n)))
            blocks.append(b[:n.value])
            active.append(a[:n.value])
            if n.value < cap:
                break
        return np.concatenate(blocks), np.concatenate(active)

    def block_totals(self, n_blocks: int) -> tuple[np.ndarray, np.ndarray]:
        s = np.zeros(n_blocks, np.int64)
        a = np.zeros(n_blocks, np.int64)
        self._c(self.lib.ls_block_totals(self.handle, _ptr(s), _ptr(a)))
        return s, a

    def block_cycles(self, n_blocks: int) -> np.ndarray:
        c = np.zeros(n_blocks, np.int64)
        self._c(self.lib.ls_block_cycles(self.handle, _ptr(c)))
        return c

    def read_var(self, var: int, slots: int, width: int) -> np.ndarray:
        out = np.empty((slots, self.z, width), np.uint64)
        self._c(self.lib.ls_read_var(self.handle, var, _ptr(out), out.nbytes))
        return out

    def read_pointers(self, var: int) -> np.ndarray:
        out = np.empty(self.z, np.int64)
        self._c(self.lib.ls_read_pointers(self.handle, var, _ptr(out), self.z))
        return out

    def read_pc_stack(self) -> np.ndarray:
        out = np.empty((self.depth + 1, self.z), np.int32)
        self._c(self.lib.ls_read_pc_stack(self.handle, _ptr(out), out.size))
        return out.astype(np.int64)

    def lane_traces(self) -> list[np.ndarray]:
        cap = self.lane_trace_cap
        blocks = np.empty((self.z, cap), np.int32)
        lens = np.empty(self.z, np.int32)
        self._c(self.lib.ls_lane_trace_fetch(self.handle, _ptr(blocks), _ptr(lens), cap))
        if (lens > cap).any():
            raise ValueError(f"lane trace truncated: raise lane_trace_cap above {int(lens.max())}")
        return [blocks[i, :lens[i]].copy() for i in range(self.z)]

    def group_traces(self) -> list[np.ndarray]:
        """Warp engine: every group's step records (block | active << 16), in step order."""
        cap, groups = self.group_trace_cap, self.groups
        recs = np.empty((groups, cap), np.int32)
        lens = np.empty(groups, np.int32)
        self._c(self.lib.ls_group_trace_fetch(self.handle, _ptr(recs), _ptr(lens), cap))
        if (lens > cap).any():
            raise ValueError(f"group trace truncated: raise group_trace_cap above {int(lens.max())}")
        return [recs[g, :lens[g]].copy() for g in range(groups)]

    def sync(self) -> None:
        self._c(self.lib.ls_machine_sync(self.handle))

    def __del__(self):
        if getattr(self, "handle", None):
            self.lib.ls_machine_destroy(self.handle)
            self.handle = None


def _as_i64(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a).astype(np.int64))


def rng_uniform(key: np.ndarray, counter: np.ndarray) -> np.ndarray:
    """Device evaluation of runtime.rng_uniform (keys/counters cast like numpy astype)."""
    k, c = np.broadcast_arrays(_as_i64(key), _as_i64(counter))
    k, c = np.ascontiguousarray(k), np.ascontiguousarray(c)
    out = np.empty(k.shape, np.float64)
    _check(load().ls_rng_uniform(_ptr(k), _ptr(c), k.size, _ptr(out)))
    return out


def target_eval(target, which: str, x: np.ndarray) -> np.ndarray:
    from .workloads import TARGET_GAUSSIAN

    x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
    z = x.shape[0]
    if target.kind == TARGET_GAUSSIAN:
        params, n, norm = target.params["prec"], target.dim, target.params["norm"]
    else:
        params, n, norm = target.params["sx"], target.params["sx"].shape[0], 0.0
    params = np.ascontiguousarray(params, dtype=np.float64)
    w = 0 if which == "logpdf" else 1
    out = np.empty(z if w == 0 else (z, target.dim), np.float64)
    _check(load().ls_target_eval(target.kind, w, target.dim, n, _ptr(params), norm, _ptr(x), z,
                                 _ptr(out)))
    return out
