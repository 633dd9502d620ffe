"""The C ABI library builds for sm_100a, loads on CPU and exports the header's symbols.

No compute calls here (there is no GPU on the builder); calls that need a
device must fail loudly instead of falling back to the CPU.
"""

import ctypes as C

import numpy as np
import pytest

import paper_1910_11141_b200 as L
from paper_1910_11141_b200 import _native
from paper_1910_11141_b200.lowering import BLOCK_DTYPE, OP_DTYPE, VAR_DTYPE
from conftest import has_gpu


def test_library_exports_every_header_symbol():
    lib = _native.load()
    names = _native.header_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native._SIGS), "ctypes signatures must cover the header exactly"
    assert lib.ls_abi_version() == 3


def test_struct_layouts_match_header():
    assert OP_DTYPE.itemsize == 56 and BLOCK_DTYPE.itemsize == 32 and VAR_DTYPE.itemsize == 24
    assert C.sizeof(_native.Status) == 64
    assert C.sizeof(_native.MachineOpts) == 36  # 9 int32 fields (group_trace_cap added in ABI v3)


def test_sass_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(has_gpu(), reason="checks the no-device failure mode")
def test_no_cpu_fallback_without_device():
    fib = L.compile_program(L.compile_source(L.workloads.FIBONACCI))
    with pytest.raises(L.DeviceError):
        L.run(fib, [np.array([3])], depth=8)
    with pytest.raises(L.DeviceError):
        L.runtime.rng_uniform(np.array([1]), np.array([1]))


def test_host_only_kernel_is_rejected():
    from paper_1910_11141_b200.lowering import lower
    from paper_1910_11141_b200.pc_vm import infer_types
    from paper_1910_11141_b200.runtime import F64, VType, register_kernel, words

    register_kernel("host_square", 1, lambda ins, z: ins[0] ** 2, lambda ins: ins[0])
    cp = L.compile_program(L.compile_source("def f(x) { return host_square(x); }"))
    types = infer_types(cp.flat, [F64])
    with pytest.raises(NotImplementedError, match="no CPU fallback"):
        lower(cp, types)
    assert words(VType("f64", 3)) == 3 and words(F64) == 1
