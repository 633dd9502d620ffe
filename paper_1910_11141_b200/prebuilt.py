"""Programs whose specialised (codegen) libraries are built ahead of time.

`__graft_entry__.build()` compiles these on the CPU builder so neither the
GPU tests nor `bench.py` ever invoke nvcc on the GPU box. Each entry is the
exact (program, input types, lowering options) the consumer uses, so the
content hash in codegen.library_for matches.
"""

from __future__ import annotations

import numpy as np

from .runtime import VType

F64, I64 = VType("f64"), VType("i64")


def nuts(dim: int, rho: float, entry: str = "nuts_main", **cfg):
    from . import compile_program, compile_source, correlated_gaussian, nuts_lite_source
    from .workloads import NutsConfig

    config = NutsConfig(**cfg)
    target = correlated_gaussian(dim, rho)
    cp = compile_program(compile_source(nuts_lite_source(config, target), entry))
    return config, target, cp


BENCH = dict(dim=100, rho=0.5, step_size=0.25, leaf_steps=4, max_depth=10, iterations=10)
# NUTS cases the GPU tests run through the specialised warp engine
TEST_NUTS = [
    dict(dim=2, rho=0.5, step_size=0.25, leaf_steps=4, max_depth=6, iterations=20),
    dict(dim=100, rho=0.5, step_size=0.25, leaf_steps=4, max_depth=10, iterations=3),
    dict(dim=5, rho=0.5, step_size=0.25, leaf_steps=4, max_depth=8, iterations=4),
]
# single-leaf programs (entry = leapfrog) whose fused superblock the per-step test checks
# against the reference's leapfrog vectors (tests/golden/leapfrog.npz)
LEAPFROG = [(2, 1), (2, 4), (100, 1), (100, 4)]
# BASELINE configs 3, 4 and 5 as bench.py measures them (their own bench-line objects); config 3
# runs 20 iterations: with 5 the launch is the tail of the few chains that build depth-10 trees
CONFIG3 = dict(n=1000, d=25, seed=0, step_size=0.05, leaf_steps=4, max_depth=10, iterations=20)
# BASELINE config 4: the 100k x 100 design (sx = 80 MB streams through shared memory), the
# reference's own measured setting (depth 10, step 0.004, 2 iterations)
CONFIG4 = dict(n=100_000, d=100, seed=0, step_size=0.004, leaf_steps=4, max_depth=10, iterations=2)
CONFIG5 = dict(dim=1000, rho=9999 / 10999, step_size=0.02, leaf_steps=4, max_depth=15, iterations=2)
# the headline target with dispersed starting points and a smaller step: trees of varying depth,
# so lanes of a warp diverge (the case program-counter autobatching exists for)
DISPERSED = dict(dim=100, rho=0.5, step_size=0.1, leaf_steps=4, max_depth=10, iterations=10)
# logistic-regression cases (DMMA two-GEMM gradient): gradient-only programs and one NUTS run
# (the two tall designs take the streamed path: n >= kLrStreamMinN; 20001 x 7 ends on an odd word)
LR_GRAD = [(200, 5, 7), (1000, 25, 0), (20001, 7, 3), (100_000, 100, 0)]
LR_NUTS = dict(n=200, d=5, seed=7, step_size=0.1, leaf_steps=2, max_depth=5, iterations=3)


def lr_gradient(n: int, d: int, seed: int):
    from . import compile_program, compile_source, logistic_regression

    t = logistic_regression(n, d, seed)
    return t, compile_program(compile_source(f"def gradient(w) {{ return {t.grad}(w); }}", "gradient"))


def lr_nuts(n: int, d: int, seed: int, **cfg):
    from . import compile_program, compile_source, logistic_regression, nuts_lite_source
    from .workloads import NutsConfig

    config = NutsConfig(**cfg)
    t = logistic_regression(n, d, seed)
    return config, t, compile_program(compile_source(nuts_lite_source(config, t), "nuts_main"))


def specs():
    """[(label, compiled, input types)] for every prebuilt specialised library."""
    from . import compile_program, compile_source
    from .workloads import corpus

    out = []
    for kw in [BENCH, DISPERSED, *TEST_NUTS]:
        kw = dict(kw)
        dim, rho = kw.pop("dim"), kw.pop("rho")
        _, _, cp = nuts(dim, rho, **kw)
        out.append((f"nuts_d{dim}_T{kw['iterations']}", cp, [VType("f64", dim), I64]))
    for d, steps in LEAPFROG:
        _, _, cp = nuts(d, 0.5, step_size=0.25, leaf_steps=steps, max_depth=6, iterations=1, entry="leapfrog")
        out.append((f"leapfrog_d{d}_L{steps}", cp, [VType("f64", d), VType("f64", d), VType("f64")]))
    for n, d, seed in LR_GRAD:
        _, cp = lr_gradient(n, d, seed)
        out.append((f"lr_grad_{n}x{d}", cp, [VType("f64", d)]))
    kw = dict(LR_NUTS)
    _, t, cp = lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
    out.append(("lr_nuts", cp, [VType("f64", t.dim), I64]))
    kw = dict(CONFIG3)
    _, t, cp = lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
    out.append(("config3", cp, [VType("f64", t.dim), I64]))
    kw = dict(CONFIG4)
    _, t, cp = lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
    out.append(("config4", cp, [VType("f64", t.dim), I64]))
    kw = dict(CONFIG5)
    dim, rho = kw.pop("dim"), kw.pop("rho")
    _, _, cp = nuts(dim, rho, **kw)
    out.append(("config5", cp, [VType("f64", dim), I64]))
    for e in corpus():
        cp = compile_program(compile_source(e.source, e.entry))
        ins = e.make_inputs(np.random.default_rng(0), 2)
        from .runtime import vtype_of

        out.append((e.name, cp, [vtype_of(a) for a in ins]))
    return out


def build_all(workers: int = 8, verbose: bool = False) -> list:
    """Compile every prebuilt specialised library (in parallel); returns their paths."""
    from concurrent.futures import ThreadPoolExecutor

    from . import codegen
    from .lowering import lower
    from .pc_vm import infer_types

    dps = [lower(cp, infer_types(cp.flat, ts), optimize=True, superblocks=True) for _, cp, ts in specs()]
    # longest compiles first (ptxas time grows with the program's op count and DMMA
    # call sites): the pool's makespan is then close to total / workers
    dps.sort(key=lambda dp: -(len(dp.ops) + 400 * sum(t.kind == 2 for t in dp.targets)))
    with ThreadPoolExecutor(workers) as ex:
        paths = list(ex.map(lambda dp: codegen.library_for(dp, verbose=verbose), dps))
    keep = {p.name for p in paths}
    for stale in codegen.GEN_DIR.glob("liblockstep_b200_*.so"):  # drop libraries of older sources
        if stale.name not in keep:
            stale.unlink()
    for hdr in codegen.GEN_DIR.glob("gen_*.cuh"):
        if f"liblockstep_b200_{hdr.stem[4:]}.so" not in keep:
            hdr.unlink()
    return paths
