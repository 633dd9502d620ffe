"""Shared fixtures. `-m gpu` tests need a B200 and call the CUDA VM through the C ABI;
everything else runs on CPU (host pipeline, oracle vs golden fixtures, ABI loading,
gloo multi-process tests)."""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a VM")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """Make sure the in-tree CUDA library exists (nvcc cross-compiles on CPU too)."""
    from paper_1910_11141_b200 import build

    if not build.is_current():
        build.build()


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "golden.json").read_text())


def load_npz(name: str):
    return np.load(GOLDEN / name)


@pytest.fixture(scope="session")
def corpus_compiled():
    import paper_1910_11141_b200 as L

    out = {}
    for e in L.corpus():
        cfg = L.compile_source(e.source, e.entry)
        out[e.name] = (e, cfg, L.compile_program(cfg))
    return out


def oracle_run(prog, inputs, depth, **kw):
    """Run the CPU oracle (test infrastructure) on a compiled program."""
    import paper_1910_11141_b200 as L
    from oracle import lockstep_oracle as O
    from paper_1910_11141_b200.pc_vm import infer_types
    from paper_1910_11141_b200.runtime import vtype_of

    types = infer_types(prog.flat, [vtype_of(np.asarray(a)) for a in inputs])
    return O.run(prog, inputs, depth=depth, types=types,
                 targets=L.workloads.device_targets(), **kw)


def nuts_program(meta_case: dict, entry: str = "nuts_main"):
    import paper_1910_11141_b200 as L

    t = L.correlated_gaussian(meta_case["dim"], meta_case["rho"])
    cfg = L.NutsConfig(**meta_case["config"])
    return cfg, t, L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), entry))


def split_lanes(lens: np.ndarray, flat: np.ndarray) -> list[np.ndarray]:
    offs = np.concatenate([[0], np.cumsum(lens)])
    return [flat[offs[i]:offs[i + 1]].astype(np.int64) for i in range(len(lens))]


def has_gpu() -> bool:
    try:
        from paper_1910_11141_b200 import _native

        return _native.device_count() > 0
    except Exception:  # noqa: BLE001
        return False


os.environ.setdefault("PYTHONHASHSEED", "0")
