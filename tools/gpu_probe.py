"""Quick device-vs-oracle probe over the corpus and a few NUTS configs (dev tool)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_11141_b200 as L  # noqa: E402
from oracle import lockstep_oracle as O  # noqa: E402
from paper_1910_11141_b200.pc_vm import infer_types  # noqa: E402
from paper_1910_11141_b200.runtime import vtype_of  # noqa: E402


def oracle(prog, ins, depth):
    types = infer_types(prog.flat, [vtype_of(a) for a in ins])
    return O.run(prog, ins, depth=depth, types=types,
                 targets=L.workloads.device_targets(), lane_traces=True)


def main():
    rng = np.random.default_rng(1)
    for e in L.corpus():
        prog = L.compile_program(L.compile_source(e.source, e.entry))
        for z in (1, 7, 32):
            ins = e.make_inputs(rng, z)
            for opt in (False, True):
                got, tr = L.run(prog, ins, depth=64, optimize=opt)
                ref = oracle(prog, ins, 64)
                ok_out = (got.tobytes() == ref.output.tobytes()) if got.dtype.kind != "f" else \
                    np.allclose(got, ref.output, rtol=1e-12, atol=0)
                ok_tr = [s.active for s in tr.steps] == [a for _, a in ref.steps]
                print(f"{e.name:10s} z={z:3d} opt={opt}: out={ok_out} trace={ok_tr} "
                      f"steps={tr.step_count}/{len(ref.steps)}", flush=True)
    for d, depth_cap, iters in ((2, 6, 20), (5, 10, 5), (100, 10, 3)):
        cfg = L.NutsConfig(step_size=0.25, leaf_steps=4, max_depth=depth_cap, iterations=iters)
        t = L.correlated_gaussian(d, 0.5)
        prog = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, t), "nuts_main"))
        z = 64
        q0 = np.zeros((z, d))
        key = np.random.default_rng(0).integers(0, 2**31, z).astype(np.int64)
        t0 = time.time()
        got, tr, m = L.run(prog, [q0, key], depth=cfg.min_stack_depth, lane_trace_cap=200000,
                           return_machine=True)
        t1 = time.time()
        ref = oracle(prog, [q0, key], cfg.min_stack_depth)
        err = np.max(np.abs(got - ref.output) / np.maximum(np.abs(ref.output), 1e-300))
        lt = m.lane_traces()
        same_lanes = all(np.array_equal(lt[i], ref.lane_blocks[i]) for i in range(z))
        print(f"nuts d={d}: max rel err {err:.3e}, trace equal "
              f"{[s.active for s in tr.steps] == [a for _, a in ref.steps]}, lane traces {same_lanes}, "
              f"device {t1 - t0:.3f}s", flush=True)
        # multi-group throughput mode
        z2 = 4096
        q0 = np.zeros((z2, d))
        key = np.random.default_rng(1).permutation(2**31)[:z2].astype(np.int64) if False else \
            np.arange(z2, dtype=np.int64) * 7919 + 11
        for sched in ("min_pc", "most_populated"):
            t0 = time.time()
            got2, tr2 = L.run(prog, [q0, key], depth=cfg.min_stack_depth, lanes_per_group=128,
                              schedule=sched)
            t1 = time.time()
            print(f"  z={z2} sched={sched}: {t1 - t0:.3f}s util={L.utilization(tr2, {t.grad}):.3f} "
                  f"grads={tr2.useful_invocations({t.grad})}", flush=True)
        sub = slice(0, 64)
        ref2 = oracle(prog, [q0[sub], key[sub]], cfg.min_stack_depth)
        err2 = np.max(np.abs(got2[sub] - ref2.output) / np.maximum(np.abs(ref2.output), 1e-300))
        print(f"  multi-group first 64 lanes vs oracle: max rel err {err2:.3e}", flush=True)


if __name__ == "__main__":
    main()
