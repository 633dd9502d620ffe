"""Mint golden fixtures from the reference implementation (run in the builder container).

Imports the UNMODIFIED reference package from /root/reference/pkg/src (read
only) and records, with the numpy/OpenBLAS build of this container:

* rng_uniform known answers over a key x counter grid     (runtime.py:288-303)
* `(a*b).sum(axis=1)` results for many row lengths       (runtime.py:248-250)
* gaussian logpdf (einsum order) for several dims        (workloads.py:188-189)
* flat IR text of every corpus program and NUTS configs  (compiler.py:510-538)
* outputs, step traces and stack-op counts of pc_vm.run on the corpus
* NUTS chains, global traces and per-lane block sequences
* single-leaf leapfrog vectors (entry='leapfrog')         (test_acceptance.py:294-312)
* logistic-regression logpdf/grad values                  (workloads.py:216-228)
* local-static engine schedules + gradient utilisation     (local_exec.py:142-193)
* long runs for the in-distribution checks: the reference's own chains (samples) of a
  5-d correlated gaussian and of logistic regression 200x5, plus the reference's moment
  ground truth (reference_moments / moment_fn, workloads.py:126-128, 230-249)

The GPU box has no /root/reference; tests read only these files.
Usage: python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import platform
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import lockstep as R  # noqa: E402
from lockstep import ir as Rir  # noqa: E402
from lockstep.runtime import rng_uniform  # noqa: E402

OUT = Path(__file__).resolve().parent

NUTS_CASES = [
    # name, dim, rho, NutsConfig kwargs, z, key seed
    ("nuts_d2", 2, 0.5, dict(step_size=0.25, leaf_steps=4, max_depth=6, iterations=20), 64, 0),
    ("nuts_d5", 5, 0.5, dict(step_size=0.25, leaf_steps=4, max_depth=10, iterations=5), 32, 1),
    ("nuts_d100", 100, 0.5, dict(step_size=0.25, leaf_steps=4, max_depth=10, iterations=3), 16, 0),
    ("nuts_d3m", 3, -0.2, dict(step_size=0.125, leaf_steps=3, max_depth=8, iterations=6), 24, 7),
    # the benchmarked configuration (bench.py / prebuilt.BENCH): 100-d, T=10, depth 10
    ("nuts_d100_T10", 100, 0.5, dict(step_size=0.25, leaf_steps=4, max_depth=10, iterations=10), 64, 0),
]

# local-static engine (Alg. 1, reference local_exec.py) vs the pc VM: gradient utilisation
# (reference test_acceptance.py:236-266 runs the first two)
LOCAL_CASES = [
    # name, dim, rho, NutsConfig kwargs, z, key seed
    ("util_z30", 2, 0.5, dict(step_size=0.25, leaf_steps=4, max_depth=6, iterations=12, seed=0), 30, 3),
    ("util_z1", 2, 0.5, dict(step_size=0.25, leaf_steps=4, max_depth=6, iterations=12, seed=0), 1, 3),
    ("util_d5_z64", 5, 0.5, dict(step_size=0.1, leaf_steps=4, max_depth=8, iterations=6, seed=0), 64, 11),
]


def env() -> dict:
    import numpy

    cfg = {}
    try:
        cfg = {k: str(v) for k, v in numpy.show_config(mode="dicts").get("Build Dependencies", {})
               .get("blas", {}).items()}
    except Exception:  # noqa: BLE001
        pass
    return {"numpy": numpy.__version__, "python": platform.python_version(),
            "machine": platform.machine(), "blas": cfg}


def rng_grid() -> dict:
    keys = np.array([0, 1, 7, 42, 123456789, 2**31 - 1, 2**31, -5, -(2**40), 2**62], np.int64)
    ctrs = np.array([0, 1, 2, 3, 17, 100, 1048576, 2**33 + 5], np.int64)
    kk, cc = np.meshgrid(keys, ctrs, indexing="ij")
    kk, cc = kk.ravel(), cc.ravel()
    u = rng_uniform(kk, cc)
    # float counters (integral and fractional) hash as int64 after truncation
    fc = np.array([0.0, 3.0, 3.7, 1e6 + 0.5, 2.0**40], np.float64)
    kf = np.full(fc.shape, 7, np.int64)
    uf = rng_uniform(kf, fc)
    return {"keys": kk, "ctrs": cc, "u": u, "fkeys": kf, "fctrs": fc, "fu": uf}


def dot_rows() -> dict:
    rng = np.random.default_rng(99)
    ns = [1, 2, 3, 7, 8, 9, 15, 16, 17, 100, 127, 128, 129, 200, 255, 256, 257, 300, 503, 1000, 2500]
    a_all, b_all, lens, res = [], [], [], []
    for n in ns:
        for _ in range(3):
            a = rng.normal(size=(1, n)) * rng.choice([1e-3, 1.0, 1e3])
            b = rng.normal(size=(1, n))
            res.append(R.runtime.resolve_kernel("dot").fn((a, b), 1)[0])
            a_all.append(a[0])
            b_all.append(b[0])
            lens.append(n)
    return {"lens": np.array(lens), "a": np.concatenate(a_all), "b": np.concatenate(b_all),
            "res": np.array(res)}


def einsum_cases() -> dict:
    out = {}
    rng = np.random.default_rng(3)
    for d in (2, 5, 25, 100, 128):
        t = R.correlated_gaussian(d, 0.5)
        x = rng.normal(size=(4, d))
        lp = R.runtime.resolve_kernel(t.logpdf).fn((x,), 4)
        cov = np.full((d, d), 0.5)
        np.fill_diagonal(cov, 1.0)
        out[f"x{d}"] = x
        out[f"lp{d}"] = lp
        out[f"P{d}"] = np.linalg.inv(cov)
        out[f"g{d}"] = R.runtime.resolve_kernel(t.grad).fn((x,), 4)
    return out


def corpus_runs() -> tuple[dict, dict]:
    arrays, meta = {}, {}
    rng = np.random.default_rng(2024)
    for e in R.corpus():
        cfg = R.compile_source(e.source, e.entry)
        cp = R.compile_program(cfg)
        meta[e.name] = {"ir": Rir.print_ir(cp.flat), "classes": cp.classes, "runs": []}
        for z in (1, 7, 32):
            ins = e.make_inputs(rng, z)
            out, tr = R.pc_vm.run(cp, ins, depth=64)
            tag = f"{e.name}_z{z}"
            for k, a in enumerate(ins):
                arrays[f"{tag}_in{k}"] = a
            arrays[f"{tag}_out"] = out
            meta[e.name]["runs"].append({
                "z": z, "tag": tag, "n_inputs": len(ins),
                "steps": [[s.block, s.active] for s in tr.steps],
                "stack_ops": tr.stack_ops,
            })
    return arrays, meta


def nuts_runs() -> tuple[dict, dict]:
    arrays, meta = {}, {}
    for name, d, rho, kw, z, seed in NUTS_CASES:
        t = R.correlated_gaussian(d, rho)
        cfg = R.NutsConfig(**kw)
        src = R.nuts_lite_source(cfg, t)
        cp = R.compile_program(R.compile_source(src, "nuts_main"))
        q0 = np.zeros((z, d))
        key = np.random.default_rng(seed).integers(0, 2**31, z).astype(np.int64)
        lanes = [[] for _ in range(z)]

        def obs(m, b, sel, lanes=lanes):
            for lane in np.flatnonzero(sel):
                lanes[lane].append(b)

        out, tr = R.pc_vm.run(cp, [q0, key], depth=cfg.min_stack_depth, observer=obs)
        arrays[f"{name}_key"] = key
        arrays[f"{name}_out"] = out
        arrays[f"{name}_lane_len"] = np.array([len(x) for x in lanes], np.int32)
        arrays[f"{name}_lane_blocks"] = np.concatenate([np.array(x, np.int16) for x in lanes])
        arrays[f"{name}_steps"] = np.array([[Rir_index(cp, s.block), s.active] for s in tr.steps],
                                           np.int32)
        meta[name] = {"dim": d, "rho": rho, "config": kw, "z": z, "key_seed": seed,
                      "target": t.name, "ir": Rir.print_ir(cp.flat), "stack_ops": tr.stack_ops,
                      "useful_grads": int(sum(s.active * s.prims.get(t.grad, 0) for s in tr.steps))}
    return arrays, meta


def local_runs() -> tuple[dict, dict]:
    """trace_local (reference local_exec.py:188-193) and pc_vm.run on the same batch: the
    local engine's schedule, outputs and both gradient utilisations (metrics.py:52-76)."""
    from lockstep.local_exec import trace_local
    from lockstep.metrics import utilization

    arrays, meta = {}, {}
    for name, d, rho, kw, z, seed in LOCAL_CASES:
        t = R.correlated_gaussian(d, rho)
        cfg = R.NutsConfig(**kw)
        src = R.nuts_lite_source(cfg, t)
        cg = R.compile_source(src, "nuts_main")
        cp = R.compile_program(cg)
        q0 = np.zeros((z, d))
        key = np.random.default_rng(seed).integers(0, 2**31, size=z).astype(np.int64)
        lout, lt = trace_local(cg, [q0, key])
        pout, pt = R.pc_vm.run(cp, [q0, key], depth=cfg.min_stack_depth)
        counted = {t.grad}
        arrays[f"{name}_key"] = key
        arrays[f"{name}_local_out"] = lout
        arrays[f"{name}_pc_out"] = pout
        labels = sorted({s.block for s in lt.steps})
        arrays[f"{name}_local_steps"] = np.array(
            [[labels.index(s.block), s.active, s.prims.get(t.grad, 0)] for s in lt.steps], np.int32)
        meta[name] = {"dim": d, "rho": rho, "config": kw, "z": z, "key_seed": seed, "target": t.name,
                      "local_labels": labels,
                      "util_local": utilization(lt, counted), "util_pc": utilization(pt, counted),
                      "pc_step_count": pt.step_count, "local_step_count": lt.step_count}
    return arrays, meta


# in-distribution cases: name, target factory, NutsConfig kwargs, z, key seed
DIST_CASES = [
    ("dist_g5", lambda: R.correlated_gaussian(5, 0.9),
     dict(step_size=0.2, leaf_steps=4, max_depth=8, iterations=200, seed=0), 128, 5),
    ("dist_lr200x5", lambda: R.logistic_regression(200, 5, seed=7),
     dict(step_size=0.1, leaf_steps=4, max_depth=8, iterations=150, seed=0), 64, 6),
]


def dist_runs() -> tuple[dict, dict]:
    """Long reference runs (pc_vm.run from q0 = 0): the chains themselves (workloads.py:477
    chain_array layout) and the target's moment ground truth, for distribution checks of
    device runs on other seeds (tests/test_distribution.py)."""
    arrays, meta = {}, {}
    for name, make, kw, z, seed in DIST_CASES:
        t = make()
        cfg = R.NutsConfig(**kw)
        cp = R.compile_program(R.compile_source(R.nuts_lite_source(cfg, t), "nuts_main"))
        key = np.random.default_rng(seed).integers(0, 2**31, size=z).astype(np.int64)
        out, tr = R.pc_vm.run(cp, [np.zeros((z, t.dim)), key], depth=cfg.min_stack_depth)
        arrays[f"{name}_key"] = key
        arrays[f"{name}_samples"] = R.workloads.chain_array(out, cfg, t.dim)
        mean, cov = t.reference_moments()
        arrays[f"{name}_mean"], arrays[f"{name}_cov"] = np.asarray(mean), np.asarray(cov)
        meta[name] = {"dim": t.dim, "config": kw, "z": z, "key_seed": seed, "target": t.name,
                      "useful_grads": int(sum(s.active * s.prims.get(t.grad, 0) for s in tr.steps))}
    return arrays, meta


def Rir_index(cp, label: str) -> int:
    return cp.labels.index(label)


def leapfrog_vectors() -> dict:
    out = {}
    rng = np.random.default_rng(101)
    for d, L in ((2, 1), (2, 4), (100, 1), (100, 4)):
        t = R.correlated_gaussian(d, 0.5)
        cfg = R.NutsConfig(step_size=0.25, leaf_steps=L, max_depth=6, iterations=1)
        cp = R.compile_program(R.compile_source(R.nuts_lite_source(cfg, t), "leapfrog"))
        q = rng.normal(size=(8, d))
        p = rng.normal(size=(8, d))
        e = rng.choice([0.25, -0.25, 0.1], size=8)
        res, _ = R.pc_vm.run(cp, [q, p, e], depth=4)
        out[f"d{d}_L{L}_q"], out[f"d{d}_L{L}_p"], out[f"d{d}_L{L}_e"] = q, p, e
        out[f"d{d}_L{L}_out"] = res
    return out


def logreg_values() -> dict:
    out = {}
    rng = np.random.default_rng(5)
    for n, d, seed in ((25, 3, 2), (200, 5, 7), (1000, 25, 0)):
        t = R.logistic_regression(n, d, seed)
        w = rng.normal(size=(6, d)) * 0.5
        tag = f"lr{n}x{d}s{seed}"
        out[f"{tag}_w"] = w
        out[f"{tag}_lp"] = R.runtime.resolve_kernel(t.logpdf).fn((w,), 6)
        out[f"{tag}_g"] = R.runtime.resolve_kernel(t.grad).fn((w,), 6)
    return out


def main():
    if sys.argv[1:] == ["dist"]:  # only the long runs (a few minutes), merged into golden.json
        meta = json.loads((OUT / "golden.json").read_text())
        arrays, meta["dist"] = dist_runs()
        np.savez_compressed(OUT / "dist_runs.npz", **arrays)
        (OUT / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
        print("wrote dist fixtures to", OUT)
        return
    meta = {"env": env(), "generator": "tests/golden/make_golden.py",
            "reference": "/root/reference/pkg/src/lockstep"}
    np.savez_compressed(OUT / "rng_kat.npz", **rng_grid())
    np.savez_compressed(OUT / "dot_rows.npz", **dot_rows())
    np.savez_compressed(OUT / "gauss_logpdf.npz", **einsum_cases())
    arrays, cmeta = corpus_runs()
    np.savez_compressed(OUT / "corpus_runs.npz", **arrays)
    meta["corpus"] = cmeta
    arrays, nmeta = nuts_runs()
    np.savez_compressed(OUT / "nuts_runs.npz", **arrays)
    meta["nuts"] = nmeta
    arrays, lmeta = local_runs()
    np.savez_compressed(OUT / "local_runs.npz", **arrays)
    meta["local"] = lmeta
    np.savez_compressed(OUT / "leapfrog.npz", **leapfrog_vectors())
    np.savez_compressed(OUT / "logreg.npz", **logreg_values())
    arrays, meta["dist"] = dist_runs()
    np.savez_compressed(OUT / "dist_runs.npz", **arrays)
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print("wrote fixtures to", OUT)


if __name__ == "__main__":
    main()
