#!/usr/bin/env python
"""Headline benchmark: NUTS gradient evaluations / s on the B200 program-counter VM.

Workload (BASELINE.json configs[1], the chain-count sweep's headline point):
NUTS-lite on the 100-d equicorrelated gaussian (rho=0.5, target g100p500),
max_tree_depth 10, step 0.25, 4 leapfrog steps per leaf, fp64, 2^16 chains
per GPU, T iterations per step. A "step" runs the whole sampler program
for every chain (all T iterations) — one pass of the hot path over one
batch. Synthetic inputs: q0 = 0, unique per-chain keys.

Metric unit: useful gradient evaluations, counted exactly as the reference
does (sum over VM steps of active lanes x grad invocations in the block;
reference metrics.py:68-76) — 2L per leaf per chain.

Arms:
  default            the B200 VM (this repo), chains sharded over ranks (weak scaling)
  --impl reference   the reference's CPU algorithm (the oracle port of pc_vm.run),
                     rank 0 only, on the host cores, bounded sample per step

Timing: per step, CUDA events around the VM launch on the machine's stream
(the library records them: ls_status.kernel_ms); W untimed warm-up steps;
L2 flushed between timed steps; max over ranks. `e2e` times the public API
call `paper_1910_11141_b200.run` with host arrays (H2D + D2H inside).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NUTS gradient evals/sec vs #chains at 1/2/4/8 B200 (+ % of roofline)"
UNIT = "grad_evals/s"
FP64_PEAK_FALLBACK = 37.0  # TFLOP/s, tools/fp64_peaks.cu on this pool's B200 (DFMA 36.9, DMMA 37.0)
FP32_PEAK_FALLBACK = 2250.0 / 2 / 3  # 3xTF32: nominal dense bf16 / 2 (TF32) / 3 MMAs per product


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--chains", type=int, default=1 << 16, help="chains per GPU")
    ap.add_argument("--config4-chains", type=int, default=1 << 13, help="config-4 line: chains")
    ap.add_argument("--config5-chains", type=int, default=1 << 16, help="config-5 line: chains")
    ap.add_argument("--dim", type=int, default=100)
    ap.add_argument("--iterations", type=int, default=10)
    ap.add_argument("--depth", type=int, default=10)
    ap.add_argument("--engine", default="warp", choices=("warp", "cta"),
                    help="warp: 32-lane group per warp + DMMA + superblocks; cta: CTA groups")
    ap.add_argument("--lanes", type=int, default=128, help="lanes per CTA group (cta engine)")
    ap.add_argument("--groups", type=int, default=0, help="persistent CTAs (0 = auto)")
    ap.add_argument("--exact-logpdf", action="store_true",
                    help="numpy einsum summation order for logpdf (default: DMMA form, 1e-15 rel)")
    ap.add_argument("--schedule", default="priority", choices=("min_pc", "most_populated", "local", "priority"),
                    help="block selection (paper_1910_11141_b200/schedule.py); lanes never depend on it")
    ap.add_argument("--no-codegen", action="store_true",
                    help="warp engine with the op interpreter instead of specialised block code")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-chains", type=int, default=256)
    ap.add_argument("--no-sweep", action="store_true", help="skip the 2^10..2^20 chain sweep")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32 (tcgen05) arm")
    ap.add_argument("--no-configs", action="store_true", help="skip BASELINE configs 3, 4 and 5")
    ap.add_argument("--cpu-iterations", type=int, default=10)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def program(args):
    import paper_1910_11141_b200 as L

    cfg = L.NutsConfig(step_size=0.25, leaf_steps=4, max_depth=args.depth,
                       iterations=args.iterations, seed=0)
    target = L.correlated_gaussian(args.dim, 0.5)
    cp = L.compile_program(L.compile_source(L.nuts_lite_source(cfg, target), "nuts_main"))
    return cfg, target, cp


def chain_keys(first: int, count: int) -> np.ndarray:
    """Unique per-chain keys (default_rng integers collide at 2^16+);
    a key depends only on the global chain id, so sharding does not change any chain."""
    from paper_1910_11141_b200.distributed import chain_keys as keys

    return keys(first, first + count)


class Clocks:
    """SM clock and throttle-reason sampling during the timed region (B200_PROFILING.md
    clocks line): an NVML thread every 10 ms (the timed region is a few hundred ms,
    shorter than nvidia-smi's start-up), nvidia-smi -lms as the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device: int):
        import threading

        self.samples: list[tuple[float, float, int]] = []
        self.proc = None
        self.stop_evt = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = int(vis.split(",")[device]) if vis and vis.split(",")[0].isdigit() else device
            self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.sample()  # the first sample is taken before the timed steps start
            self.thread = threading.Thread(target=self.loop, daemon=True)
            self.thread.start()
        except Exception:
            self.nv = None
            self.path = tempfile.mktemp(suffix=".csv")
            q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            try:
                self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                              "-i", str(device), "-lms", "100"],
                                             stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            except OSError:
                self.proc = None

    def sample(self) -> None:
        nv = self.nv
        self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)),
                             float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)),
                             int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))))

    def loop(self) -> None:
        while not self.stop_evt.wait(0.01):
            try:
                self.sample()
            except Exception:
                return

    def stop(self) -> dict:
        if self.nv is not None:
            self.sample()  # and one after the last timed step
            self.stop_evt.set()
            self.thread.join()
            reasons = sorted({name for name, attr in self.REASONS for _, _, bits in self.samples
                              if bits & getattr(self.nv, attr, 0)})
            return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                    "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                    "samples": len(self.samples), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = [r.split(", ") for r in open(self.path).read().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for name, val in zip(names, r[5:9]):
                if val.strip() == "Active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(rows), "source": "nvidia-smi"}


def flush_l2(torch, dev):
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    buf.fill_(1)
    torch.cuda.synchronize(dev)


def measured_traffic(lib) -> dict | None:
    """DRAM bytes per launch of this very library (by content hash) from an `ncu --set full`
    capture of the same command, recorded in profiles/traffic.json; None if not captured."""
    if lib is None:
        return None
    try:
        table = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        return None
    return table.get(os.path.basename(str(lib)))


def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(path))
    except (OSError, ValueError):
        return {}


def cpu_reference_sample(args, cfg, target, cp, chains: int, iterations: int, engine: str = "pc",
                         want_output: bool = False):
    """Time the oracle port of the reference engines on host cores: `pc` = pc_vm.run (numpy
    masked mode, reference pc_vm.py:368-383), `local` = run_local (Alg. 1, local_exec.py:142-185).
    Chains 0..chains-1 of the benchmark workload (same keys). Returns (useful grads, seconds[, out])."""
    import paper_1910_11141_b200 as L
    from oracle import lockstep_oracle as O
    from paper_1910_11141_b200.pc_vm import infer_types
    from paper_1910_11141_b200.runtime import vtype_of

    small = L.NutsConfig(step_size=cfg.step_size, leaf_steps=cfg.leaf_steps, max_depth=cfg.max_depth,
                         iterations=iterations, seed=0)
    src = L.nuts_lite_source(small, target)
    q0 = np.zeros((chains, target.dim))
    key = chain_keys(0, chains)
    if engine == "local":
        cg = L.compile_source(src, "nuts_main")
        t0 = time.perf_counter()
        out, steps = O.run_local(cg, [q0, key], targets={target.name: L.device_target(target.name)}, max_steps=None)
        dt = time.perf_counter() - t0
        grads = sum(a * g for _, a, g in steps)
        return (grads, dt, out) if want_output else (grads, dt)
    scp = L.compile_program(L.compile_source(src, "nuts_main"))
    types = infer_types(scp.flat, [vtype_of(q0), vtype_of(key)])
    t0 = time.perf_counter()
    res = O.run(scp, [q0, key], depth=small.min_stack_depth, types=types,
                targets={target.name: L.device_target(target.name)}, max_steps=None)
    dt = time.perf_counter() - t0
    grads = 0
    for b, active in res.steps:
        blk = scp.flat.blocks[b]
        grads += active * sum(1 for op in blk.ops if getattr(op, "prim", None) is not None
                              and op.prim.name == target.grad)
    return (grads, dt, res.output) if want_output else (grads, dt)


def host_info() -> dict:
    """CPU model, usable cores and the numpy / BLAS build the CPU baseline ran on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        cfg = np.show_config(mode="dicts")["Build Dependencies"]["blas"]
        blas = f"{cfg.get('name')} {cfg.get('version')}"
    except Exception:  # noqa: BLE001
        pass
    return {"cpu_model": model, "cores": len(os.sched_getaffinity(0)), "numpy": np.__version__,
            "blas": blas, "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS")}


def cpu_baseline(args, cfg, target, cp, reps: int = 5) -> tuple[dict, np.ndarray]:
    """Warm best-of-`reps` of the pc engine port plus one run_local, both on the same
    bounded sample (chains 0..cpu_chains-1 of the workload, cpu_iterations iterations)."""
    cpu_reference_sample(args, cfg, target, cp, 16, 2)  # warm: imports, numpy dispatch
    best, out = None, None
    for _ in range(reps):
        g, dt, o = cpu_reference_sample(args, cfg, target, cp, args.cpu_chains, args.cpu_iterations,
                                        want_output=True)
        if best is None or dt < best[1]:
            best, out = (g, dt), o
    gl, dtl = cpu_reference_sample(args, cfg, target, cp, args.cpu_chains, args.cpu_iterations, "local")
    info = host_info()
    return {"value": best[0] / best[1], "unit": UNIT, "cores": info["cores"], "kind": "port",
            "sample": (f"oracle port of reference pc_vm.run (numpy masked mode), {target.name}, chains "
                       f"0..{args.cpu_chains - 1} of this workload x {args.cpu_iterations} iterations: "
                       f"best of {reps} warm runs {best[1]:.2f} s"),
            "local_engine": {"value": gl / dtl, "unit": UNIT, "seconds": dtl,
                             "sample": "oracle port of reference local_exec.run_local (Alg. 1), same chains"},
            "host": info}, out


def run_reference_arm(args):
    """The reference's own algorithm on host cores (oracle port of pc_vm.run; the reference is
    pure Python/numpy and cannot travel to the GPU box), bounded sample per step."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores))
    cfg, target, cp = program(args)
    for _ in range(args.warmup):
        cpu_reference_sample(args, cfg, target, cp, min(args.cpu_chains, 64), args.cpu_iterations)
    tot_g, tot_t = 0, 0.0
    for _ in range(args.steps):
        g, dt = cpu_reference_sample(args, cfg, target, cp, args.cpu_chains, args.cpu_iterations)
        tot_g += g
        tot_t += dt
    value = tot_g / tot_t
    sample = (f"oracle port of reference pc_vm.run (numpy masked mode), {target.name}, "
              f"{args.cpu_chains} chains x {args.cpu_iterations} iterations per step")
    config = {"workload": f"NUTS-lite on {args.dim}-d correlated gaussian (rho=0.5, {target.name})",
              "chains_per_step": args.cpu_chains, "iterations": args.cpu_iterations,
              "max_tree_depth": args.depth, "step_size": 0.25, "leaf_steps": 4, "precision": "fp64",
              "engine": "oracle port of reference pc_vm.run (numpy masked mode, min-pc schedule)",
              "note": ("the same program and keys as the b200 arm's chains 0..chains_per_step-1; the "
                       "CPU cannot run the b200 arm's chain count within a bounded step")}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (q0=0, unique per-chain keys)",
        "config": config,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, target):
    return {"workload": f"NUTS-lite on {args.dim}-d correlated gaussian (rho=0.5, {target.name})",
            "chains_per_gpu": args.chains, "iterations": args.iterations, "max_tree_depth": args.depth,
            "step_size": 0.25, "leaf_steps": 4, "precision": "fp64",
            "engine": args.engine, "codegen": args.engine == "warp" and not args.no_codegen,
            "lanes_per_group": 32 if args.engine == "warp" else args.lanes,
            "schedule": args.schedule,
            "logpdf": "numpy einsum order" if args.exact_logpdf else "DMMA q.(Pq) (within 1e-15 rel)",
            "l2": "flushed between timed steps (256 MiB write); outputs exceed L2"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch

    import paper_1910_11141_b200 as L
    from paper_1910_11141_b200 import _native
    from paper_1910_11141_b200.lowering import lower
    from paper_1910_11141_b200.pc_vm import infer_types
    from paper_1910_11141_b200.runtime import vtype_of

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    cfg, target, cp = program(args)
    z = args.chains
    first = rank * z
    q0 = np.zeros((z, args.dim))
    key = chain_keys(first, z)
    types = infer_types(cp.flat, [vtype_of(q0), vtype_of(key)])
    warp = args.engine == "warp"
    dp = lower(cp, types, optimize=True, superblocks=warp)
    lib = None
    if warp and not args.no_codegen:
        from paper_1910_11141_b200 import codegen

        lib = codegen.library_for(dp)  # prebuilt by __graft_entry__.build() for the default config
    prog = _native.Program(dp, lib, device=local)  # this rank's GPU (LOCAL_RANK)
    mach = _native.MachineHandle(prog, z, cfg.min_stack_depth, sched=args.schedule,
                                 lanes_per_cta=0 if warp else args.lanes, ctas=args.groups,
                                 exact_logpdf=args.exact_logpdf, warp_groups=warp)
    from paper_1910_11141_b200.schedule import block_keys

    mach.set_block_keys(block_keys(cp.flat, cp.labels, args.schedule,
                                   np.flatnonzero(np.asarray(dp.blocks["grads"]) > 0)))
    # inputs resident in HBM before the timed region
    q0_d = torch.zeros((z, args.dim), dtype=torch.float64, device=dev)
    key_d = torch.from_numpy(key).to(dev)
    mach.set_input_device(0, q0_d.data_ptr(), q0_d.numel() * 8)
    mach.set_input_device(1, key_d.data_ptr(), key_d.numel() * 8)

    def one_step():
        mach.reset()
        st = mach.run(-1)
        if st.kind != _native.RUN_HALTED:
            raise RuntimeError(f"VM did not halt: status {st.kind}")
        return st

    for _ in range(args.warmup):
        one_step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    clocks = Clocks(local)
    times, grads, launches0 = [], 0, None
    for _ in range(args.steps):
        flush_l2(torch, dev)
        st = one_step()
        if launches0 is None:
            launches0 = st.launches - 1
        times.append(st.kernel_ms)
        grads += st.useful_grads
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    launches = st.launches - launches0
    t_total = sum(times) / 1e3
    if world > 1:
        t = torch.tensor([t_total], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        g = torch.tensor([grads], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(g)
        t_total, grads_all = float(t.item()), float(g.item())
    else:
        grads_all = float(grads)
    value = grads_all / t_total
    ms_per_step = 1e3 * t_total / args.steps

    # roofline of the dominant kernel (vm_kernel: the whole step is one launch)
    flops_per_grad = L.device_target(target.name).grad_flops
    args_leaf_steps = cfg.leaf_steps  # the superblock executes L+1 of the 2L reference gradients
    achieved = (grads / args.steps) * flops_per_grad / (np.mean(times) / 1e3) / 1e12
    traffic = measured_traffic(lib)
    roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_FALLBACK, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_FALLBACK,
                "traffic": traffic["bytes_per_launch"] if traffic else None,
                "traffic_source": traffic["source"] if traffic else "no ncu capture of this library",
                "executed_frac": achieved / FP64_PEAK_FALLBACK * (args_leaf_steps + 1) / (2 * args_leaf_steps),
                "note": ("fp64 gradient FLOPs (2*d^2 per useful, reference-equivalent grad: 2L per leaf) / "
                         "vm_kernel launch time; executed_frac counts the L+1 contractions per leaf the fused "
                         "superblock performs; peak = measured fp64 DFMA/DMMA rate (tools/fp64_peaks.cu), "
                         "MEASURED_PEAKS.json has no fp64 figure")}

    # e2e through the public API with host buffers (H2D of inputs, D2H of chains inside)
    e2e = None
    if not args.no_e2e:
        reps = max(1, min(args.steps, 3))
        g_e2e = 0
        # the first two calls are warm-up: lowering + device allocation, then the second
        # pinned output buffer (the previous result is still referenced during a call)
        for i in range(reps + 2):
            if i == 2:
                t0 = time.perf_counter()
                g_e2e = 0
            out, tr = L.run(cp, [q0, key], depth=cfg.min_stack_depth, engine=args.engine, device=local,
                            lanes_per_group=None if warp else args.lanes, groups=args.groups,
                            schedule=args.schedule, exact_logpdf=args.exact_logpdf,
                            codegen=warp and not args.no_codegen)
            g_e2e += tr.useful_invocations({target.grad})
        dt = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([dt], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            dt = float(tt.item())
            gg = torch.tensor([g_e2e], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(gg)
            g_e2e = float(gg.item())
        e2e = {"value": g_e2e / dt, "unit": UNIT, "h2d_bytes_per_step": int(q0.nbytes + key.nbytes),
               "d2h_bytes_per_step": int(out.nbytes),
               "path": "paper_1910_11141_b200.run(compiled, [q0, key]) with host numpy arrays"}

    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, cpu_out = cpu_baseline(args, cfg, target, cp)
        if args.cpu_iterations == args.iterations:
            # the CPU sample is chains 0..n-1 of this very workload: check the device's rows
            n = cpu_out.shape[0]
            dev_rows = torch.empty((n, cpu_out.shape[1]), dtype=torch.float64, device=dev)
            mach.copy_output_rows_to(dev_rows.data_ptr(), n)
            got = dev_rows.cpu().numpy()
            err = float((np.abs(got - cpu_out) / np.maximum(np.abs(cpu_out), 1.0)).max())
            parity = {"chains": int(n), "max_rel_err": err, "tolerance": 1e-9, "ok": bool(err < 1e-9),
                      "against": "the CPU baseline's oracle run of the same chains (reference pc_vm.run port)"}

    # BASELINE config 2: grad evals/s vs chains (2^10 .. 2^20) in fp64 and fp32, one warm + one
    # timed launch per point; plus the fp32 arm at this run's chain count
    sweep, fp32 = None, None
    keys_dp = np.flatnonzero(np.asarray(dp.blocks["grads"]) > 0)

    def one_point(zz, precision, reps=1):
        mz = _native.MachineHandle(prog, zz, cfg.min_stack_depth, sched=args.schedule, ctas=args.groups,
                                   exact_logpdf=args.exact_logpdf, warp_groups=warp, precision=precision)
        mz.set_block_keys(block_keys(cp.flat, cp.labels, args.schedule, keys_dp))
        qz = torch.zeros((zz, args.dim), dtype=torch.float64, device=dev)
        kz = torch.from_numpy(chain_keys(first, zz)).to(dev)
        mz.set_input_device(0, qz.data_ptr(), qz.numel() * 8)
        mz.set_input_device(1, kz.data_ptr(), kz.numel() * 8)
        mz.run(-1)
        ms, gsum = 0.0, 0
        for _ in range(reps):
            mz.reset()
            flush_l2(torch, dev)
            stz = mz.run(-1)
            ms += stz.kernel_ms
            gsum += stz.useful_grads
        del mz, qz, kz
        return gsum / (ms / 1e3), ms / reps

    flops_per_grad = L.device_target(target.name).grad_flops
    peaks = measured_peaks()
    # 3xTF32 = three TF32 MMAs per product; TF32 dense runs at half the bf16 rate
    tf32x3_peak = peaks["bf16_tflops"] / 2 / 3 if peaks.get("bf16_tflops") else FP32_PEAK_FALLBACK
    if warp and not args.no_fp32 and world == 1:
        v32, ms32 = one_point(z, "fp32", reps=max(1, min(args.steps, 3)))
        fp32 = {"value": v32, "unit": UNIT, "ms_per_step": ms32, "chains": z,
                "roofline": {"bound": "tensor", "achieved": v32 * flops_per_grad / 1e12, "peak": tf32x3_peak,
                             "unit": "TFLOP/s", "frac": v32 * flops_per_grad / 1e12 / tf32x3_peak,
                             "note": ("useful fp32 gradient FLOPs; peak = 3xTF32 rate = MEASURED_PEAKS "
                                      "bf16_tflops / 2 (TF32) / 3 (split)")},
                "arith": "fused leapfrog in float32 on tcgen05 (kind::tf32, 3xTF32), VM control in f64"}
    if rank == 0 and world == 1 and not args.no_sweep:
        sweep = {"schedule": args.schedule, "fp64": [], "fp32": []}
        for lg in range(10, 21):
            zz = 1 << lg
            for precision in (("fp64", "fp32") if warp and not args.no_fp32 else ("fp64",)):
                v, ms = one_point(zz, precision)
                peak = FP64_PEAK_FALLBACK if precision == "fp64" else tf32x3_peak
                sweep[precision].append({"chains": zz, "value": v, "ms": ms,
                                         "frac": v * flops_per_grad / 1e12 / peak})

    # BASELINE configs 3, 4 and 5 (one warm + one timed launch each, fp64, same engine/schedule)
    configs = None
    if rank == 0 and world == 1 and warp and not args.no_configs:
        configs = {}
        from paper_1910_11141_b200 import prebuilt

        def cfg_point(label, cfgx, tx, cpx, zz, inputs_fn):
            dtx = L.device_target(tx.name)
            m2 = L.init_machine(cpx, inputs_fn(zz), depth=cfgx.min_stack_depth, engine="warp", optimize=True, device=local,
                                exact_logpdf=False, codegen="cached", schedule=args.schedule)
            m2._h.run(-1)
            m2._h.reset()
            flush_l2(torch, dev)
            st2 = m2._h.run(-1)
            v = st2.useful_grads / (st2.kernel_ms / 1e3)
            configs[label] = {"chains": zz, "iterations": cfgx.iterations, "max_tree_depth": cfgx.max_depth,
                              "step_size": cfgx.step_size, "value": v, "unit": UNIT, "ms": st2.kernel_ms,
                              "useful_grads": int(st2.useful_grads), "flops_per_grad": dtx.grad_flops,
                              "frac": v * dtx.grad_flops / 1e12 / FP64_PEAK_FALLBACK, "precision": "fp64",
                              "grad_utilization": st2.useful_grads / max(st2.launched_grads, 1)}

        kw = dict(prebuilt.CONFIG3)
        c3, t3, cp3 = prebuilt.lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
        cfg_point("config3_logreg_1000x25", c3, t3, cp3, 1 << 16,
                  lambda zz: [np.zeros((zz, t3.dim)), chain_keys(0, zz)])
        kw = dict(prebuilt.DISPERSED)
        cd, td, cpd = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
        cfg_point("dispersed_init_gauss100_eps0.1", cd, td, cpd, 1 << 16,
                  lambda zz: [np.random.default_rng(1).standard_normal((zz, td.dim)), chain_keys(0, zz)])
        configs["dispersed_init_gauss100_eps0.1"]["note"] = (
            "headline target from random starts q0 ~ N(0, I), step 0.1; the equicorrelated gaussian's "
            "U-turn time barely depends on the state, so trees keep one size per iteration (config 3 "
            "is the workload whose chains diverge: see its grad_utilization)")
        kw = dict(prebuilt.CONFIG4)
        c4, t4, cp4 = prebuilt.lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
        cfg_point("config4_logreg_100000x100", c4, t4, cp4, args.config4_chains,
                  lambda zz: [np.zeros((zz, t4.dim)), chain_keys(0, zz)])
        configs["config4_logreg_100000x100"]["note"] = (
            "one GPU's shard (BASELINE shards config 4 over 2/4/8 GPUs; chains are independent, "
            "so every rank runs this workload on its own range); sx (80 MB) streams through each "
            "warp's shared-memory ring by bulk async copies")
        kw = dict(prebuilt.CONFIG5)
        c5, t5, cp5 = prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)
        cfg_point("config5_gauss1000_cond1e4_depth15", c5, t5, cp5, args.config5_chains,
                  lambda zz: [np.zeros((zz, t5.dim)), chain_keys(0, zz)])

    # cross-chain diagnostics over all ranks: the one NCCL exchange (outside the timed region)
    from paper_1910_11141_b200.distributed import diagnostics

    chains_d = torch.empty((z, args.iterations, args.dim), dtype=torch.float64, device=dev)
    mach.copy_output_to(chains_d.data_ptr(), chains_d.numel() * 8)
    diag = diagnostics(chains_d[:, args.iterations // 2:] if args.iterations >= 4 else chains_d)
    diag_summary = {"chains": diag.chains, "draws_per_chain": diag.draws,
                    "rhat_max": float(np.max(diag.rhat)), "ess_min": float(np.min(diag.ess)),
                    "mean_abs_max": float(np.max(np.abs(diag.mean))),
                    "collective": "all_reduce of split-R-hat/ESS sufficient statistics"
                                  + (" (NCCL)" if world > 1 else " (single rank)")}
    del chains_d

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (q0=0, unique per-chain keys, random-free target parameters)",
            "config": {**workload_config(args, target), "parallelism": f"chains sharded over {world} GPU(s)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk, "diagnostics": diag_summary, "parity": parity, "fp32": fp32, "sweep": sweep,
            "configs": configs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
