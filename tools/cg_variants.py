"""Build (here) or time (on the GPU) codegen variants of the bench program: dev tool.
usage: python tools/cg_variants.py build|time VAR=val,VAR=val ..."""
import os, sys, subprocess, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
variants = [dict(kv.split("=") for kv in v.split(",")) for v in sys.argv[2:]] or [{}]
if sys.argv[1] == "build":
    procs = []
    for v in variants:
        env = dict(os.environ, **v)
        code = ("import sys; sys.path.insert(0,'.'); import numpy as np; from paper_1910_11141_b200 import prebuilt, codegen;"
                "from paper_1910_11141_b200.lowering import lower; from paper_1910_11141_b200.pc_vm import infer_types;"
                "from paper_1910_11141_b200.runtime import VType;"
                "kw=dict(prebuilt.BENCH); c,t,cp=prebuilt.nuts(kw.pop('dim'), kw.pop('rho'), **kw);"
                "dp=lower(cp, infer_types(cp.flat,[VType('f64',100),VType('i64')]), optimize=True, superblocks=True);"
                "print(codegen.library_for(dp))")
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env, cwd=ROOT,
                                      stderr=subprocess.DEVNULL))
    for p in procs:
        p.wait()
else:
    for v in variants:
        env = dict(os.environ, **v)
        out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "2", "--no-e2e",
                              "--no-cpu-baseline"], env=env, cwd=ROOT, capture_output=True, text=True)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
            print(f"{v}: {d['value'] / 1e6:.1f} M grads/s, {d['ms_per_step']:.1f} ms", flush=True)
        except Exception:
            print(v, "FAILED", out.stderr[-500:], flush=True)
