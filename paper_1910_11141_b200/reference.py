"""The reference package `lockstep` — the host pipeline this engine accelerates.

The B200 engine replaces the reference's execution engine (`lockstep.pc_vm`,
reference pkg/src/lockstep/pc_vm.py) and keeps everything above it as the
reference's own code: the source language (`frontend`), the IR types (`ir`),
the compiler (`compiler.compile_program`), the NUTS-lite generator and target
densities (`workloads`), traces (`metrics`) and exceptions (`errors`). Those
modules are used unchanged, imported from an installed `lockstep`.

Lookup order: an importable `lockstep` (the drop-in setting: the user has the
reference installed), else the copy `__graft_entry__.build()` installs with
pip into `baseline/_ref/` (git-ignored; it travels with the repository
snapshot to the GPU box).
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
VENDORED = ROOT / "baseline" / "_ref"


def _load():
    try:
        return importlib.import_module("lockstep")
    except ImportError:
        pass
    if (VENDORED / "lockstep" / "__init__.py").exists():
        sys.path.insert(0, str(VENDORED))
        return importlib.import_module("lockstep")
    raise ImportError(
        "the reference package `lockstep` is not installed: `pip install` it, or run "
        "`python -c 'import __graft_entry__ as g; g.build()'`, which installs it into baseline/_ref")


lockstep = _load()
ir = importlib.import_module("lockstep.ir")
compiler = importlib.import_module("lockstep.compiler")
frontend = importlib.import_module("lockstep.frontend")
runtime = importlib.import_module("lockstep.runtime")
workloads = importlib.import_module("lockstep.workloads")
metrics = importlib.import_module("lockstep.metrics")
errors = importlib.import_module("lockstep.errors")
pc_vm = importlib.import_module("lockstep.pc_vm")

