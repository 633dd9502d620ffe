"""Program-specialised block code for the warp engine (paper §5 "static blocks").

The generic VM (`csrc/lsb_vm.cuh::exec_block`) interprets resolved op
descriptors: every op pays a descriptor read, a dispatch and operand address
arithmetic, and every scalar goes through HBM. This module partially
evaluates a lowered program (`lowering.DeviceProgram`) into CUDA source with
one function per flat block:

* operand rows, widths and stack-pointer rows become constants;
* block-local scalar temporaries become registers (never stored);
* vector ops call the fixed-width helpers of `csrc/lsb_gen_rt.cuh`;
* target contractions and the fused leapfrog superblock stay warp-cooperative
  (every thread of the warp calls them, active or not).

Semantics are exactly `exec_block<true>` (same arithmetic helpers, same
fault rules, same terminators); tests compare both paths lane for lane.

The generated header is compiled together with `csrc/engine.cu`
(`-DLSB_GENERATED=...`) into `_lib/gen/liblockstep_b200_<hash>.so`, a full
copy of the C ABI whose warp kernel dispatches to the generated blocks.
Libraries are cached by content hash; `__graft_entry__.build()` pre-builds the
benchmark program so nothing compiles on the GPU box.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
from pathlib import Path

import numpy as np

from . import build as _build
from .lowering import DeviceProgram
from .runtime import OPCODES

GEN_DIR = _build.LIB_DIR / "gen"
OP = {v: k for k, v in OPCODES.items()}
F64, I64, BOOL = 0, 1, 2
STACKED, REGISTER, TEMPORARY = 0, 1, 2
PUSH, UPDATE, POP = 0, 1, 2
# code-shape switches (part of the generated text, hence of the library hash)
OPT = {"noalias": os.environ.get("LSB_CG_NOALIAS", "0") == "1",
       "spcache": os.environ.get("LSB_CG_SPCACHE", "1") == "1",
       "staged": os.environ.get("LSB_CG_STAGED", "0") == "1",
       # B-fragment register double-buffering in mtile_gemm
       "bpf": int(os.environ.get("LSB_CG_BPF", "0")),
       # loads in flight per thread in the generated vector loops
       "ewu": int(os.environ.get("LSB_CG_EWU", "16")),
       # dev-only superblock phase clocks (tools/sb_profile.py)
       "sbprof": int(os.environ.get("LSB_CG_SBPROF", "0")),
       # blocks with identical code on different variables share warp steps (find_pairs)
       "pairs": int(os.environ.get("LSB_CG_PAIRS", "1")),
       # warps per CTA of the warp engine (registers per thread = 65536 / (32 * wmax))
       "wmax": int(os.environ.get("LSB_CG_WMAX", "16")),
       # dev-only per-block SM-cycle accounting (clock64 + atomics; tools/block_profile.py)
       "bprof": int(os.environ.get("LSB_CG_BPROF", "0")),
       # n-tiles per superblock kick pass
       "lfkc": int(os.environ.get("LSB_CG_LFKC", "2")),
       # shared out-of-line vector helpers instead of a loop per call site
       "ool": int(os.environ.get("LSB_CG_OOL", "0")),
       # blocks with more ops than this run on the (i-cache resident) op interpreter:
       # straight-line code for e.g. draw_normals' 1300 ops misses the i-cache on
       # every fetch (0 = always generate)
       "interp_min": int(os.environ.get("LSB_CG_INTERP_MIN", "0")),
       # hoist constant-index element reads of unwritten storage to the segment start
       "hoist": int(os.environ.get("LSB_CG_HOIST", "1")),
       # fuse `t = x +- y` into the one or two dots that consume it
       "ewdot": int(os.environ.get("LSB_CG_EWDOT", "1")),
       # one pass for several copies of the same source
       "fanout": int(os.environ.get("LSB_CG_FANOUT", "1")),
       # block functions inlined into the dispatcher (no call ABI) or out of line
       "inline": int(os.environ.get("LSB_CG_INLINE", "1")),
       # the superblock inlined into its block too
       "sbinline": int(os.environ.get("LSB_CG_SBINLINE", "1")),
       # warp_gauss (DMMA grad / fast logpdf) inlined at its call sites
       "wginline": int(os.environ.get("LSB_CG_WGINLINE", "0"))}


def _block_qual() -> str:
    return "__forceinline__" if OPT["inline"] else "__noinline__"


def _u64(bits: int) -> str:
    return f"0x{int(bits) & 0xFFFFFFFFFFFFFFFF:016x}ull"


class _Gen:
    def __init__(self, dp: DeviceProgram):
        self.dp = dp
        self.opt = dict(OPT)  # per generator: generation may run on several threads
        self.vars = dp.vars
        off, stk = 0, {}
        for v in range(len(dp.vars)):
            if dp.vars[v]["cls"] == STACKED:
                stk[v] = off
                off += int(dp.vars[v]["width"])
        self.stk = stk
        self.flat = int(dp.flat_rows)
        self.in_seg = False
        self.dirty: set[int] = set()
        self.cache: set[int] = set()
        self.cached_vars: set[int] = set()
        self.pre: list[str] = []
        self.pm: dict[int, int] | None = None  # paired block: var of block A -> var of block B
        self.pair_ops = None                   # ... and block B's ops (per-lane immediates)

    # ---- operand access -----------------------------------------------------------------
    def w(self, v):
        return int(self.vars[v]["width"])

    def cls(self, v):
        return int(self.vars[v]["cls"])

    def local(self, v, locals_):
        return v in locals_

    def imm0(self, k, op) -> str:
        """imm0 of op k as an expression (a paired block's vslice may differ per lane)."""
        a = int(op["imm0"])
        if self.pm is not None and self.pair_ops is not None:
            bb = int(self.pair_ops[k]["imm0"])
            if bb != a:
                return f"(sB_ ? {bb} : {a})"
        return str(a)

    def _pair(self, v):
        """The partner block's variable at v's position (paired blocks), or None."""
        if self.pm is None:
            return None
        u = self.pm.get(v, v)
        return None if u == v else u

    def _base1(self, v):
        if self.cls(v) == STACKED:
            return f"({self.flat} + D * {self.stk[v]})"
        return str(int(self.vars[v]["row"]))

    def base(self, v):
        """Row expression of the variable's slot 0 (per lane in a paired block)."""
        u = self._pair(v)
        if u is None or self._base1(u) == self._base1(v):
            return self._base1(v)
        return f"(sB_ ? {self._base1(u)} : {self._base1(v)})"

    def spr(self, v):
        """Stack-pointer row expression of stacked variable v (per lane in a paired block)."""
        r = int(self.vars[v]["sp"])
        u = self._pair(v)
        if u is None or int(self.vars[u]["sp"]) == r:
            return str(r)
        return f"(sB_ ? {int(self.vars[u]['sp'])} : {r})"

    def vid(self, v):
        """Variable id expression for fault reports."""
        u = self._pair(v)
        return str(v) if u is None else f"(sB_ ? {u} : {v})"

    def ptr(self, v):
        """Pointer expression to the variable's current top (read)."""
        if self.cls(v) == STACKED:
            r = int(self.vars[v]["sp"])
            if self.in_seg:  # stack pointer cached in a register for the segment
                return f"ln.row({self.base(v)} + (sp{r} > 0 ? sp{r} - 1 : 0) * {self.w(v)})"
            return f"ln.top({self.base(v)}, {self.spr(v)}, {self.w(v)})"
        return f"ln.row({self.base(v)})"

    def disjoint(self, dv, act, sv, d_off, s_off, w):
        """Can a copy of w words from sv(+s_off) to dv(+d_off) use the no-alias helper?"""
        if self.pm is not None:  # must hold for both blocks of a pair
            pm, self.pm = self.pm, None
            try:
                return (self.disjoint(dv, act, sv, d_off, s_off, w) and
                        self.disjoint(pm.get(dv, dv), act, pm.get(sv, sv), d_off, s_off, w))
            finally:
                self.pm = pm
        if dv == sv:
            return act == PUSH  # a push writes a fresh slot above the top it reads
        if self.cls(dv) == STACKED or self.cls(sv) == STACKED:
            return True  # distinct variables: stack regions never overlap other storage
        d0 = int(self.vars[dv]["row"]) + d_off
        s0 = int(self.vars[sv]["row"]) + s_off
        return d0 + w <= s0 or s0 + w <= d0

    def same_rows(self, dv, act, sv, d_off, s_off):
        """Statically the same storage (an in-place chain link): the copy is a no-op."""
        if self.pm is not None:  # must hold for both blocks of a pair
            pm, self.pm = self.pm, None
            try:
                return (self.same_rows(dv, act, sv, d_off, s_off) and
                        self.same_rows(pm.get(dv, dv), act, pm.get(sv, sv), d_off, s_off))
            finally:
                self.pm = pm
        if act == PUSH:
            return False
        if self.cls(dv) == STACKED or self.cls(sv) == STACKED:
            return dv == sv and d_off == s_off
        return int(self.vars[dv]["row"]) + d_off == int(self.vars[sv]["row"]) + s_off

    def copy(self, w, dst_expr, src_expr, dv, act, sv, d_off=0, s_off=0):
        if self.same_rows(dv, act, sv, d_off, s_off):
            return "  /* in place */"
        if self.opt["staged"] and w >= 16:
            return f"  copy_staged<{w}>({dst_expr}, {src_expr}, sm);"
        fn = "copy_nr" if self.opt["noalias"] and self.disjoint(dv, act, sv, d_off, s_off, w) else "copy"
        return f"  {fn}<{w}>({dst_expr}, {src_expr});"

    def scalar(self, v, locals_):
        if v in locals_:
            return f"s{v}"
        if self.cls(v) == REGISTER and self.w(v) == 1:
            # register scalars are loaded once per segment and reused until written
            if v not in self.cache:
                self.pre.append(f"r{v} = {self.ptr(v)}[0];")
                self.cache.add(v)
                self.cached_vars.add(v)
            return f"r{v}"
        return f"{self.ptr(v)}[0]"

    # ---- one op -------------------------------------------------------------------------------
    def op_code(self, k, op, locals_, pos):
        """C++ statements for one non-cooperative op (inside `if (ok)`)."""
        self.pre = []
        lines = self._op_code(k, op, locals_, pos)
        out = int(op["out"])
        self.cache.discard(out)
        return self.pre + lines

    def _op_code(self, k, op, locals_, pos):
        opc = int(op["opcode"])
        act = int(op["action"])
        out = int(op["out"])
        nin = int(op["nin"])
        ins = [int(x) for x in op["in"][:nin]]
        name = OP.get(opc, "?")
        lines = []
        if act == POP:
            sp = int(self.vars[out]["sp"])
            if not self.in_seg:
                return [f"{{ int& s_ = ln.sp_row({self.spr(out)});",
                        f"  if (s_ < 1) {{ f = StepFault{{{pos}, LS_RUN_UNDERFLOW, {self.vid(out)}, 0}}; ok = false; goto {self.end}; }}",
                        "  --s_; }"]
            self.dirty.add(sp)
            lines += [f"if (sp{sp} < 1) {{ f = StepFault{{{pos}, LS_RUN_UNDERFLOW, {self.vid(out)}, 0}}; ok = false; goto {self.end}; }}",
                      f"--sp{sp};"]
            return lines
        width = int(op["width"])
        fk = int(op["kind"]) == F64
        S = lambda j: self.scalar(ins[j], locals_)  # noqa: E731
        P = lambda j: self.ptr(ins[j])  # noqa: E731
        W = lambda j: self.w(ins[j])  # noqa: E731
        # scalar expression forms
        expr = None
        if name == "const":
            expr = _u64(op["bits"])
        elif name == "id" and width == 1:
            expr = S(0)
        elif name in ("add", "sub", "mul", "div", "min", "max") and width == 1:
            x, y = S(0), S(1)
            if fk:
                fn = {"add": "__dadd_rn", "sub": "__dsub_rn", "mul": "__dmul_rn", "div": "__ddiv_rn"}.get(name)
                expr = (f"f64_bits({fn}(as_f64({x}), as_f64({y})))" if fn else
                        f"f_min({x}, {y}, {'true' if name == 'min' else 'false'})")
            else:
                expr = {"add": f"({x} + {y})", "sub": f"({x} - {y})",
                        "mul": f"(uint64_t)((unsigned long long)({x}) * (unsigned long long)({y}))",
                        "div": f"i64_div({x}, {y})",
                        "min": f"i_min({x}, {y}, true)", "max": f"i_min({x}, {y}, false)"}[name]
        elif name in ("le", "lt", "eq"):
            x, y = S(0), S(1)
            c = {"le": "<=", "lt": "<", "eq": "=="}[name]
            if fk:
                expr = f"(uint64_t)(as_f64({x}) {c} as_f64({y}))"
            elif name == "eq":
                expr = f"(uint64_t)({x} == {y})"
            else:
                expr = f"(uint64_t)((int64_t)({x}) {c} (int64_t)({y}))"
        elif name in ("and", "or"):
            c = "&&" if name == "and" else "||"
            expr = f"(uint64_t)(({S(0)} != 0) {c} ({S(1)} != 0))"
        elif name == "not":
            expr = f"(uint64_t)({S(0)} == 0)"
        elif name == "neg" and width == 1:
            expr = f"f64_bits(-as_f64({S(0)}))" if fk else f"(0ull - {S(0)})"
        elif name == "abs" and width == 1:
            expr = f"f64_bits(fabs(as_f64({S(0)})))" if fk else f"i_abs({S(0)})"
        elif name in ("sqrt", "exp", "log", "sin", "cos", "floor") and width == 1:
            # transcendental bodies are shared out-of-line calls: straight-line blocks
            # with many of them (draw_normals) would otherwise overflow the i-cache
            fn = {"sqrt": "__dsqrt_rn", "floor": "floor"}.get(name, f"ool_{name}")
            expr = f"f64_bits({fn}(as_f64({S(0)})))"
        elif name == "select" and width == 1:
            expr = f"(({S(0)} != 0) ? {S(1)} : {S(2)})"
        elif name == "vget":
            expr = (f"({P(0)})[clip(to_i64({S(1)}, {str(self.vars[ins[1]]['kind'] == F64).lower()}), "
                    f"{W(0)}) * S]")
        elif name == "vslice" and width == 1:
            expr = f"({P(0)})[{self.imm0(k, op)} * S]"
        elif name == "vfill" and width == 1:
            expr = S(0)
        elif name == "rng_uniform":
            kf = str(self.vars[ins[0]]["kind"] == F64).lower()
            cf = str(self.vars[ins[1]]["kind"] == F64).lower()
            expr = (f"ool_rng(to_i64({S(0)}, {kf}), to_i64({S(1)}, {cf}))" if self.opt["ool"] else
                    f"f64_bits(lsb::rng_uniform(to_i64({S(0)}, {kf}), to_i64({S(1)}, {cf})))")
        elif name == "dot":
            expr = f"f64_bits(dot<{W(0)}>({P(0)}, {P(1)}))"
        elif name == "logpdf":
            expr = f"f64_bits(target_logpdf(a.targets[{int(op['imm0'])}], {P(0)}, S, a.exact_logpdf))"

        if expr is not None and out in locals_:
            return [f"s{out} = {expr};"]
        # memory destination
        dst, post = self.dst(out, act, width, pos)
        lines += dst
        if name == "alloc":  # unobserved save: allocate the slot, copy nothing
            return lines + ["  (void)d_;"] + post + ["}"]
        if name == "normals":
            kf = str(self.vars[ins[0]]["kind"] == F64).lower()
            return lines + [f"  normals_lane(d_, S, to_i64({S(0)}, {kf}), as_f64({S(1)}), {int(op['imm0'])}, "
                            f"{int(op['imm1'])});"] + post + ["}"]
        if expr is not None:
            lines.append(f"  d_[0] = {expr};")
        elif name == "id":
            lines.append(self.copy(width, "d_", P(0), out, act, ins[0]))
        elif name == "vslice":
            lo = self.imm0(k, op)
            if lo.isdigit():
                lines.append(self.copy(width, "d_", f"{P(0)} + {lo} * S", out, act, ins[0], 0, int(lo)))
            else:  # per-lane window offset (paired blocks): a plain copy
                lines.append(f"  copy<{width}>(d_, {P(0)} + {lo} * S);")
        elif name == "vcat":
            wa = W(0)
            lines.append(self.copy(wa, "d_", P(0), out, act, ins[0]))
            lines.append(self.copy(width - wa, f"d_ + {wa} * S", P(1), out, act, ins[1], wa, 0))
        elif name == "vfill":
            lines.append(f"  fill<{width}>(d_, {S(0)});")
        elif name == "vstore":
            kf = str(self.vars[ins[1]]["kind"] == F64).lower()
            lines.append(f"  {{ const uint64_t v_ = {S(2)}; const int64_t k_ = clip(to_i64({S(1)}, {kf}), {width});")
            lines.append("  " + self.copy(width, "d_", P(0), out, act, ins[0]).strip() + " d_[k_ * S] = v_; }")
        elif name == "axpy":
            lines.append(f"  axpy<{width}>(d_, as_f64({S(0)}), {P(1)}, {P(2)});")
        elif name == "select":
            lines.append(f"  select<{width}>(d_, {S(0)} != 0, {P(1)}, {P(2)});")
        elif name in ("add", "sub", "mul", "div", "min", "max"):
            xs, ys = P(0), P(1)
            if fk:
                fn = {"add": "__dadd_rn", "sub": "__dsub_rn", "mul": "__dmul_rn", "div": "__ddiv_rn"}.get(name)
                body = (f"f64_bits({fn}(as_f64(xs_[i * S]), as_f64(ys_[i * S])))" if fn else
                        f"f_min(xs_[i * S], ys_[i * S], {'true' if name == 'min' else 'false'})")
            else:
                body = {"add": "xs_[i * S] + ys_[i * S]", "sub": "xs_[i * S] - ys_[i * S]",
                        "mul": "(uint64_t)((unsigned long long)xs_[i * S] * (unsigned long long)ys_[i * S])",
                        "div": "i64_div(xs_[i * S], ys_[i * S])",
                        "min": "i_min(xs_[i * S], ys_[i * S], true)",
                        "max": "i_min(xs_[i * S], ys_[i * S], false)"}[name]
            code = {"add": 0, "sub": 1, "mul": 2, "div": 3}.get(name)
            if self.opt["ool"] and fk and code is not None:
                lines.append(f"  binop_f64_n(d_, {xs}, {ys}, {width}, {code});")
            else:
                lines.append(f"  {{ const uint64_t* xs_ = {xs}; const uint64_t* ys_ = {ys};")
                lines.append(f"    ew<{width}>(d_, [&](int i) {{ return {body}; }}); }}")
        elif name in ("neg", "abs", "sqrt", "exp", "log", "sin", "cos", "floor"):
            if fk:
                fn = {"neg": None, "abs": "fabs", "sqrt": "__dsqrt_rn", "floor": "floor"}.get(name, f"ool_{name}")
                body = "f64_bits(-as_f64(xs_[i * S]))" if name == "neg" else f"f64_bits({fn}(as_f64(xs_[i * S])))"
            else:
                body = "0ull - xs_[i * S]" if name == "neg" else "i_abs(xs_[i * S])"
            lines.append(f"  {{ const uint64_t* xs_ = {P(0)}; ew<{width}>(d_, [&](int i) {{ return {body}; }}); }}")
        elif name == "grad":
            lines.append(f"  target_grad(a.targets[{int(op['imm0'])}], {P(0)}, S, d_);")
        else:
            raise NotImplementedError(f"codegen: opcode {opc} ({name})")
        lines += post
        lines.append("}")
        return lines

    def dst(self, out, act, width, pos):
        """Open a `{ uint64_t* d_ = ...;` scope with stack checks; returns (lines, closing lines)."""
        if self.cls(out) != STACKED:
            return [f"{{ uint64_t* d_ = ln.row({self.base(out)});"], []
        sp = int(self.vars[out]["sp"])
        vo = self.vid(out)
        if self.in_seg:  # stack pointer cached in the segment's register sp<row>
            if act == PUSH:
                self.dirty.add(sp)
                return ([f"{{ if (sp{sp} >= D) {{ f = StepFault{{{pos}, LS_RUN_OVERFLOW, {vo}, 0}}; ok = false; goto {self.end}; }}",
                         f"  uint64_t* d_ = ln.row({self.base(out)} + sp{sp} * {width});"],
                        [f"  ++sp{sp};"])
            return ([f"{{ if (sp{sp} < 1) {{ f = StepFault{{{pos}, LS_RUN_UNDERFLOW, {vo}, 1}}; ok = false; goto {self.end}; }}",
                     f"  uint64_t* d_ = ln.row({self.base(out)} + (sp{sp} - 1) * {width});"], [])
        if act == PUSH:
            return ([f"{{ int& sp_ = ln.sp_row({self.spr(out)});",
                     f"  if (sp_ >= D) {{ f = StepFault{{{pos}, LS_RUN_OVERFLOW, {vo}, 0}}; ok = false; goto {self.end}; }}",
                     f"  uint64_t* d_ = ln.row({self.base(out)} + sp_ * {width});"],
                    ["  ++sp_;"])
        return ([f"{{ const int sp_ = ln.sp_row({self.spr(out)});",
                 f"  if (sp_ < 1) {{ f = StepFault{{{pos}, LS_RUN_UNDERFLOW, {vo}, 1}}; ok = false; goto {self.end}; }}",
                 f"  uint64_t* d_ = ln.row({self.base(out)} + (sp_ - 1) * {width});"], [])

    def leapfrog_fn(self, t: int) -> str:
        """The superblock instance for target slot t (its n-tile count is static here)."""
        nt = (int(self.dp.targets[t].dim) + 7) // 8
        return f"warp_leapfrog_nt<{nt}>" if nt <= 16 else "warp_leapfrog"

    def coop_code(self, op, locals_, pos):
        """A warp-cooperative op: every thread calls it; `ok` lanes participate."""
        opc = int(op["opcode"])
        name = OP.get(opc)
        out = int(op["out"])
        ins = [int(x) for x in op["in"][:int(op["nin"])]]
        if name == "leapfrog":
            bits = int(op["bits"])
            gv = bits & 0xFFFFFFFF
            gv = -1 if gv == 0xFFFFFFFF else gv
            iv = bits >> 32
            iv = -1 if iv in (0xFFFFFFFF, -1) else iv
            grow = self.base(gv) if gv >= 0 else "-1"
            irow = self.base(iv) if iv >= 0 else "-1"
            lines = ["{ ROp lf_{};"]
            for j, v in enumerate(ins[:3]):  # q, p (maybe forwarded stacked sources), e
                sp = int(self.vars[v]["sp"]) if self.cls(v) == STACKED else -1
                lines.append(f"  lf_.in_row[{j}] = {self.base(v)}; lf_.in_sp[{j}] = {sp}; lf_.in_w[{j}] = {self.w(v)};")
            return lines + [
                f"  lf_.out_row = {self.base(out)}; lf_.kind = {int(op['kind'])};",
                f"  lf_.pad = {self.base((int(op['kind']) >> 1) - 1) if int(op['kind']) >> 1 else -1};",
                f"  lf_.imm0 = {int(op['imm0'])}; lf_.imm1 = {int(op['imm1'])}; lf_.imm2 = {int(op['imm2'])};",
                f"  lf_.bits = (long long)(((unsigned long long)({grow}) & 0xffffffffull) | ((unsigned long long)({irow}) << 32));",
                f"  {self.leapfrog_fn(int(op['imm0']))}(a, ln, lf_, ok, sm, chain); }}",
            ]
        # gaussian grad / logpdf through DMMA
        act = int(op["action"])
        want_lp = name == "logpdf"
        lines = ["{ bool part_ = ok; uint64_t* cd_ = nullptr;"]
        if out in locals_:
            raise NotImplementedError("cooperative op into a register-local scalar")
        lines.append("  if (part_) {")
        d, post = self.dst(out, act, int(op["width"]), pos)
        # reuse dst() but without goto: faults here only clear part_
        d = [s.replace(f"ok = false; goto {self.end};", "ok = false; part_ = false;") for s in d]
        lines += ["    " + s for s in d]
        lines.append("    if (part_) cd_ = d_; }")
        lines.append("  }")
        x = self.ptr(ins[0])
        call = (f"  warp_gauss(a.targets[{int(op['imm0'])}], staged_B(a, {int(op['imm0'])}), part_, part_ ? (const uint64_t*){x} : nullptr, cd_, "
                f"{'true' if want_lp else 'false'}, sm, a.lf_smem_per_warp);")
        if self.dp.targets[int(op["imm0"])].kind == 2:  # logistic regression: fused DMMA pass
            t = int(op["imm0"])
            cond = f"!a.exact_logpdf && lr_coop(a, a.targets[{t}])" if want_lp else f"lr_coop(a, a.targets[{t}])"
            nt2 = (int(self.dp.targets[t].dim) + 7) // 8
            lp_ = 'true' if want_lp else 'false'
            # wide designs (NT2 >= 8): the streamed body inlined for this target's NT2 — as an
            # out-of-line call its 2·NT2 accumulators spill (config 4: 1.7x faster inlined);
            # narrow ones keep the call (config 3 at NT2 = 4 measured 2x slower inlined)
            if 8 <= nt2 <= 16:
                lines.append(f"  if ({cond} && lr_streams(a.targets[{t}], a.lf_smem_per_warp)) {{ __syncwarp(); "
                             f"warp_lr_stream_body<{nt2}, {lp_}>(a.targets[{t}], part_, "
                             f"part_ ? (const uint64_t*){x} : nullptr, cd_, sm); __syncwarp(); }}")
                cond = "else if (" + cond + ")"
            else:
                cond = "if (" + cond + ")"
            lines.append(f"  {cond} {{ __syncwarp(); warp_lr(a.targets[{t}], part_, "
                         f"part_ ? (const uint64_t*){x} : nullptr, cd_, sm, {lp_}, a.lf_smem_per_warp); "
                         "__syncwarp(); }")
            if want_lp:
                lines.append(f"  else if (part_) cd_[0] = f64_bits(target_logpdf(a.targets[{t}], {x}, S, 1));")
            else:
                lines.append(f"  else if (part_) target_grad(a.targets[{t}], {x}, S, cd_);")
        elif want_lp and int(op["bits"]) > 0:  # computed by the preceding superblock (fast mode)
            lines.append(f"  if (!a.exact_logpdf) {{ if (part_) cd_[0] = ln.row({self.base(int(op['bits']) - 1)})[0]; }}")
            lines.append(f"  else if (part_) cd_[0] = f64_bits(target_logpdf(a.targets[{int(op['imm0'])}], {x}, S, 1));")
        elif want_lp:
            lines.append("  if (!a.exact_logpdf) { __syncwarp();" + call.strip() + " __syncwarp(); }")
            lines.append(f"  else if (part_) cd_[0] = f64_bits(target_logpdf(a.targets[{int(op['imm0'])}], {x}, S, 1));")
        else:
            lines.append("  __syncwarp();")
            lines.append(call)
            lines.append("  __syncwarp();")
        if post:  # push: advance the stack pointer of participating lanes
            sp = int(self.vars[out]["sp"])
            lines.append(f"  if (part_) ++ln.sp_row({sp});")
        lines.append("}")
        return lines

    def is_coop(self, op):
        name = OP.get(int(op["opcode"]))
        if name == "leapfrog":
            return True
        if name in ("grad", "logpdf"):
            t = self.dp.targets[int(op["imm0"])]
            # gaussian grad/logpdf; logistic-regression grad/logpdf (fused DMMA, d <= 128)
            return t.kind == 1 or (t.kind == 2 and (t.dim + 7) // 8 <= 16)
        return False

    def ew_dot_fusions(self, ops, i, j, locals_, blk) -> dict[int, list[str]]:
        """`T = x (+|-) y` (f64 vector temporary, 8 <= width <= 128) consumed only by one or
        two `dot(T, a)` of this segment: one pass computes both dots without storing T
        (ew_dot; e.g. NUTS-lite's U-turn check `dq = sub(qp, qm); dot(dq, pm); dot(dq, pp)`).
        Returns {op index: lines} — the first dot emits the fused pass, the elementwise op
        and the second dot emit nothing."""
        out_lines: dict[int, list[str]] = {}
        cond = int(blk["cond"]) if int(blk["term"]) == 1 else -1

        def rows(v):
            if self.cls(v) == STACKED:
                return None
            r0 = int(self.vars[v]["row"])
            return r0, r0 + max(1, self.w(v))

        def clobbers(op, v):
            """Does op (possibly) change the storage v is read from?"""
            out, act = int(op["out"]), int(op["action"])
            if self.cls(v) == STACKED:
                return out == v  # a write, push or pop of v itself moves or changes its top
            if act == POP or self.cls(out) == STACKED:
                return False
            ro, rv = rows(out), rows(v)
            return ro[0] < rv[1] and rv[0] < ro[1]

        for k in range(i, j):
            op = ops[k]
            name = OP.get(int(op["opcode"]))
            if name not in ("add", "sub") or int(op["action"]) != UPDATE or int(op["kind"]) != F64:
                continue
            t, w = int(op["out"]), int(op["width"])
            if not (8 <= w <= 128) or t in locals_ or self.cls(t) != TEMPORARY or t == cond:
                continue
            x, y = int(op["in"][0]), int(op["in"][1])
            users = [m for m in range(len(ops)) if m != k and int(ops[m]["action"]) != POP
                     and t in [int(z) for z in ops[m]["in"][:int(ops[m]["nin"])]]]
            if not users or len(users) > 2 or any(m < k or m >= j for m in users):
                continue
            if any(int(ops[m]["out"]) == t for m in range(k + 1, len(ops))):
                continue
            dots = []
            for m in users:
                u = ops[m]
                ins = [int(z) for z in u["in"][:int(u["nin"])]]
                if OP.get(int(u["opcode"])) != "dot" or int(u["out"]) not in locals_ or ins.count(t) != 1:
                    break
                dots.append((m, ins[1] if ins[0] == t else ins[0], int(u["out"])))
            else:
                last = dots[-1][0]
                srcs = [x, y] + [a for _, a, _ in dots]
                if any(clobbers(ops[q], v) for q in range(k + 1, last) for v in srcs):
                    continue
                if any(t == a for _, a, _ in dots):
                    continue
                two = len(dots) == 2
                a1 = self.ptr(dots[0][1])
                a2 = self.ptr(dots[1][1]) if two else a1
                code = 0 if name == "add" else 1
                lines = ["{ double r1_, r2_;",
                         f"  ew_dot<{w}, {code}, {'true' if two else 'false'}>({self.ptr(x)}, {self.ptr(y)}, {a1}, {a2}, r1_, r2_);",
                         f"  s{dots[0][2]} = f64_bits(r1_);"]
                if two:
                    lines.append(f"  s{dots[1][2]} = f64_bits(r2_);")
                lines.append("}")
                out_lines[k] = []
                out_lines[dots[0][0]] = lines
                if two:
                    out_lines[dots[1][0]] = []
        return out_lines

    def copy_fanouts(self, ops, i, j, busy: set[int]) -> dict[int, list[str]]:
        """Copies of one source (same variable, offset and width) into several flat
        destinations in a segment — `id`, `vslice` and the parts of a `vcat` — become one
        pass that loads each element once (copy_fan), emitted at the first copy; e.g.
        NUTS-lite's `qm = q; qp = q; prop = q` and the leaf pack (q1, p1 three and two
        times). Moving a later write up is allowed only when nothing in between touches
        its destination or changes the source. Returns {op index: replacement lines}."""
        units = []  # [k, part, dst row, src var, src offset, width]
        for k in range(i, j):
            if k in busy:
                continue
            op = ops[k]
            name, act, out = OP.get(int(op["opcode"])), int(op["action"]), int(op["out"])
            if act != UPDATE or self.cls(out) == STACKED:
                continue
            w = int(op["width"])
            ins = [int(x) for x in op["in"][:int(op["nin"])]]
            r0 = int(self.vars[out]["row"])
            if name == "id" and w > 1 and not self.same_rows(out, act, ins[0], 0, 0):
                units.append((k, 0, r0, ins[0], 0, w))
            elif name == "vslice" and w > 1 and not self.same_rows(out, act, ins[0], 0, int(op["imm0"])):
                units.append((k, 0, r0, ins[0], int(op["imm0"]), w))
            elif name == "vcat":
                wa = self.w(ins[0])
                if wa > 1 and not self.same_rows(out, act, ins[0], 0, 0):
                    units.append((k, 0, r0, ins[0], 0, wa))
                if w - wa > 1 and not self.same_rows(out, act, ins[1], wa, 0):
                    units.append((k, 1, r0 + wa, ins[1], 0, w - wa))
        groups: dict[tuple, list] = {}
        for u in units:
            groups.setdefault((u[3], u[4], u[5]), []).append(u)

        def span(v, off, w):
            if self.cls(v) == STACKED:
                return None
            r0 = int(self.vars[v]["row"]) + off
            return r0, r0 + w

        def touches(o, lo, hi, reads=True):
            """o writes (or, with reads, also reads) flat rows [lo, hi)."""
            vs = [int(o["out"])] if int(o["action"]) != POP else []
            if reads:
                vs += [int(x) for x in o["in"][:int(o["nin"])]]
            for v in vs:
                sp = span(v, 0, max(1, self.w(v)))
                if sp is not None and sp[0] < hi and lo < sp[1]:
                    return True
            return False

        handled: dict[tuple[int, int], bool] = {}
        emit: dict[int, list[str]] = {}
        for (src, off, w), us in groups.items():
            if len(us) < 2:
                continue
            ss = span(src, off, w)
            first = us[0][0]
            keep = [us[0]]
            for u in us[1:]:
                lo, hi = u[2], u[2] + w
                if ss is not None and ss[0] < hi and lo < ss[1]:
                    continue  # destination overlaps the source
                between = ops[first + 1:u[0]]  # strictly between the group's first copy and u
                if any(touches(o, lo, hi) for o in between):
                    continue
                if ss is None:
                    if any(int(o["out"]) == src for o in between):
                        continue
                elif any(touches(o, ss[0], ss[1], reads=False) for o in between):
                    continue
                keep.append(u)
            if len(keep) < 2:
                continue
            src_expr = self.ptr(src) + (f" + {off} * S" if off else "")
            dsts = ", ".join(f"ln.row({u[2]})" for u in keep)
            emit.setdefault(first, []).extend([f"{{ uint64_t* const d_[{len(keep)}] = {{{dsts}}};",
                                               f"  copy_fan<{w}, {len(keep)}>({src_expr}, d_); }}"])
            for u in keep:
                handled[(u[0], u[1])] = True
        out_lines: dict[int, list[str]] = {}
        for u in units:  # ops with a handled part are replaced; their other parts copy here
            k = u[0]
            if not any(handled.get((k, part)) for part in (0, 1)):
                continue
            lines = out_lines.setdefault(k, list(emit.get(k, [])))
            if not handled.get((u[0], u[1])):
                src_expr = self.ptr(u[3]) + (f" + {u[4]} * S" if u[4] else "")
                lines.append(f"copy<{u[5]}>(ln.row({u[2]}), {src_expr});")
        for k, lines in emit.items():
            out_lines.setdefault(k, lines)
        return out_lines

    def hoistable_loads(self, ops, i, j, locals_) -> dict[int, str]:
        """Scalar element reads `s = vget(v, const)` of flat storage, issued together
        right after the last write of that storage in the segment (or at its start),
        so their memory latencies overlap instead of alternating with the stores
        that consume them (e.g. the 100 `chain = vstore(chain, base + k, vget(q, k))`
        of the chain store). Returns {op index: (emit-before index, line)}."""
        consts, defs = {}, {}
        written: dict[int, tuple[int, int]] = {}
        for k, op in enumerate(ops):
            if int(op["action"]) == POP:
                continue
            out = int(op["out"])
            defs[out] = defs.get(out, 0) + 1
            if OP.get(int(op["opcode"])) == "const" and int(op["kind"]) == I64:
                consts[out] = int(op["bits"])
            if self.cls(out) != STACKED:
                r0 = int(self.vars[out]["row"])
                written[k] = (r0, r0 + max(1, int(op["width"])))
        out_lines = {}
        for k in range(i, j):
            op = ops[k]
            if OP.get(int(op["opcode"])) != "vget" or int(op["action"]) != UPDATE:
                continue
            out, src, idx = int(op["out"]), int(op["in"][0]), int(op["in"][1])
            if out not in locals_ or self.cls(src) == STACKED or idx not in consts or defs.get(idx) != 1:
                continue
            if defs.get(out) != 1:
                continue
            r0 = int(self.vars[src]["row"])
            r1 = r0 + self.w(src)
            h = i  # just after the last write of the source rows before k in this segment
            for w in range(i, k):
                if w in written and written[w][0] < r1 and r0 < written[w][1]:
                    h = w + 1
            if h >= k:
                continue
            e = min(max(consts[idx], 0), self.w(src) - 1)
            out_lines[k] = (h, f"s{out} = ln.row({r0})[{e} * S];")
        # sliding window: a load is issued at most kWindow hoisted loads ahead of its use
        # (hoisting all of e.g. 100 element reads at once spills them to local memory)
        window = 16
        ks = sorted(out_lines)
        for m in range(window, len(ks)):
            h, line = out_lines[ks[m]]
            out_lines[ks[m]] = (max(h, ks[m - window] + 1), line)
        return out_lines

    def block_ops(self, b):
        blk = self.dp.blocks[b]
        return self.dp.ops[int(blk["op_begin"]):int(blk["op_begin"]) + int(blk["op_count"])]

    def pair_map(self, a, b) -> dict[int, int] | None:
        """Variable correspondence when blocks a and b are the same code on different storage
        (op by op: opcode, action, width, immediates, operand classes and widths; terminator
        kind), e.g. the two direction variants of NUTS-lite's tree calls and landing pads.
        Such a pair runs in one warp step, each lane on its own block's variables."""
        ba, bb = self.dp.blocks[a], self.dp.blocks[b]
        if int(ba["term"]) != int(bb["term"]) or int(ba["op_count"]) != int(bb["op_count"]):
            return None
        if int(ba["grads"]) or int(bb["grads"]):
            return None
        pm: dict[int, int] = {}

        def match(u, v):
            if pm.get(u, v) != v or self.cls(u) != self.cls(v) or self.w(u) != self.w(v):
                return False
            if self.dp.types[self.dp.var_names[u]] != self.dp.types[self.dp.var_names[v]]:
                return False
            pm[u] = v
            return True

        alloc_a, alloc_b = [], []
        for x, y in zip(self.block_ops(a), self.block_ops(b)):
            if self.is_coop(x) or self.is_coop(y):
                return None
            # a vslice may take its window at a different offset in each block (per-lane offset)
            fields = ("opcode", "action", "nin", "kind", "width", "imm2", "bits")
            if OP.get(int(x["opcode"])) != "vslice":
                fields += ("imm0", "imm1")
            for f in fields:
                if int(x[f]) != int(y[f]):
                    return None
            if OP.get(int(x["opcode"])) == "alloc":  # matched as sets below
                alloc_a.append(int(x["out"]))
                alloc_b.append(int(y["out"]))
                continue
            if not match(int(x["out"]), int(y["out"])):
                return None
            for j in range(int(x["nin"])):
                if not match(int(x["in"][j]), int(y["in"][j])):
                    return None
        if int(ba["term"]) == 1 and not match(int(ba["cond"]), int(bb["cond"])):
            return None
        # An alloc only reserves one slot on its variable's stack, so a block's allocs are an
        # unordered set: block B's save of (qm, qp) around a call on (qm, pm) is block A's save
        # of (qp, qm) around a call on (qp, pp). Variables the data ops left unmapped take a
        # free partner of the same storage (identity first) so the allocs map onto B's set.
        images = set(pm.values())
        for u in alloc_a:
            if u in pm:
                continue
            for v in ([u] if u in alloc_b else []) + alloc_b:
                if v not in images and match(u, v):
                    images.add(v)
                    break
            else:
                return None
        if sorted(pm[u] for u in alloc_a) != sorted(alloc_b):
            return None
        if len(set(pm.values())) != len(pm):  # a bijection of variables
            return None
        return pm

    def find_pairs(self) -> dict[int, int]:
        """Disjoint block pairs that can share a warp step (block -> partner)."""
        n = len(self.dp.blocks)
        out: dict[int, int] = {}
        if not self.opt["pairs"]:
            return out
        sig = {}
        for b in range(n):
            ops = self.block_ops(b)
            key = (int(self.dp.blocks[b]["term"]), tuple((int(o["opcode"]), int(o["width"])) for o in ops))
            sig.setdefault(key, []).append(b)
        for group in sig.values():
            for i, a in enumerate(group):
                if a in out:
                    continue
                # empty blocks (landing pads) pair only with a pad of the same successors
                empty = not len(self.block_ops(a))
                for b2 in group[i + 1:]:
                    if empty and any(int(self.dp.blocks[a][f]) != int(self.dp.blocks[b2][f]) for f in ("a", "b")):
                        continue
                    if b2 not in out and self.pair_map(a, b2) is not None:
                        out[a], out[b2] = b2, a
                        break
        return out

    def block(self, b, partner: int | None = None):
        blk = self.dp.blocks[b]
        ops = self.dp.ops[int(blk["op_begin"]):int(blk["op_begin"]) + int(blk["op_count"])]
        self.pm = self.pair_map(b, partner) if partner is not None else None
        if partner is not None and self.pm is None:
            raise AssertionError("not a block pair")
        if self.pm is not None:
            saved_opt = {k: self.opt[k] for k in ("hoist", "ewdot", "fanout")}
            self.opt.update(hoist=0, ewdot=0, fanout=0)  # their static row reasoning is per block
            self.pair_ops = self.block_ops(partner)
            try:
                return self._block(b, blk, ops, partner)
            finally:
                self.opt.update(saved_opt)
                self.pm = None
                self.pair_ops = None
        return self._block(b, blk, ops, None)

    def _block(self, b, blk, ops, partner):
        if self.opt["interp_min"] and len(ops) > self.opt["interp_min"] and partner is None:
            return (f"__device__ {_block_qual()} bool gb_{b}(const VMArgs& a, const Lane ln, bool active, "
                    f"long long chain, StepFault& f, double* sm, int& pc_, int& psp_) {{\n"
                    f"  int& msp_ = ln.sp_row(a.n_sp_rows - 1);  // the interpreter keeps pc state in memory\n"
                    f"  msp_ = psp_; ln.pcs[(psp_ - 1) * ln.L + ln.t] = pc_;\n"
                    f"  const bool h_ = exec_block<true>(a, ln, {b}, active, chain, f, sm);\n"
                    f"  psp_ = msp_; if (psp_ >= 1) pc_ = ln.pcs[(psp_ - 1) * ln.L + ln.t];\n"
                    f"  return h_;\n}}")
        # scalar block-local temporaries -> registers
        locals_ = set()
        for op in ops:
            if int(op["action"]) == POP:
                continue
            out = int(op["out"])
            scalar_type = self.dp.types[self.dp.var_names[out]].width == 0  # f64[1] stays in memory
            if self.cls(out) == TEMPORARY and scalar_type and not self.is_coop(op):
                locals_.add(out)
        for op in ops:  # an op that reads a coop output from memory keeps it in memory
            if self.is_coop(op):
                locals_.discard(int(op["out"]))
        body = [f"__device__ {_block_qual()} bool gb_{b}(const VMArgs& a, const Lane ln, bool active, "
                f"long long chain, StepFault& f, double* sm, int& pc_, int& psp_) {{",
                "  const int D = a.depth; (void)D; (void)sm; (void)chain;",
                "  bool ok = active;"]
        if partner is not None:
            body.append(f"  const bool sB_ = pc_ == {partner};  // this lane runs block {partner} (paired with {b})")
        if locals_:
            body.append("  uint64_t " + ", ".join(f"s{v} = 0" for v in sorted(locals_)) + ";")
        decl_at = len(body)
        self.cached_vars = set()
        self.end = "seg0_end"  # a leading cooperative op formats its checks before any segment
        all_sp: set[int] = set()
        seg = 0
        i = 0
        while i < len(ops):
            self.cache = set()  # memory may change across cooperative ops
            if self.is_coop(ops[i]):
                self.in_seg = False
                body += ["  " + s for s in self.coop_code(ops[i], locals_, i + 1)]
                i += 1
                continue
            self.end = f"seg{seg}_end"
            j = i
            while j < len(ops) and not self.is_coop(ops[j]):
                j += 1
            # stack pointers this segment touches: loaded once (in parallel), written back if moved
            rows = set()
            row_expr: dict[int, str] = {}
            for op in ops[i:j]:
                for v in [int(op["out"]), *[int(x) for x in op["in"][:int(op["nin"])]]]:
                    if self.cls(v) == STACKED:
                        rows.add(int(self.vars[v]["sp"]))
                        row_expr[int(self.vars[v]["sp"])] = self.spr(v)
            all_sp |= rows
            self.in_seg, self.dirty = self.opt["spcache"], set()
            if not self.opt["spcache"]:
                rows = set()
            body.append(f"  const bool ran{seg} = ok;")
            body.append("  if (ok) {")
            body += [f"    sp{r} = ln.sp_row({row_expr[r]});" for r in sorted(rows)]
            self.row_expr = row_expr
            hoisted = self.hoistable_loads(ops, i, j, locals_) if self.opt["hoist"] else {}
            fused = self.ew_dot_fusions(ops, i, j, locals_, blk) if self.opt["ewdot"] else {}
            if self.opt["fanout"]:
                for k, lines in self.copy_fanouts(ops, i, j, set(fused) | set(hoisted)).items():
                    fused.setdefault(k, lines)
            at: dict[int, list[str]] = {}
            for k, (h, line) in hoisted.items():
                at.setdefault(h, []).append(line)
            body += ["    " + s for s in at.get(i, [])]
            while i < j:
                if i in fused:
                    body += ["    " + s for s in fused[i]]
                elif i not in hoisted:
                    body += ["    " + s for s in self.op_code(i, ops[i], locals_, i + 1)]
                body += ["    " + s for s in at.get(i + 1, [])]
                i += 1
            body.append("  }")
            body.append(f"  {self.end}:;")
            if self.dirty:
                body.append(f"  if (ran{seg}) {{ " + " ".join(f"ln.sp_row({row_expr[r]}) = sp{r};"
                                                          for r in sorted(self.dirty)) + " }")
            self.in_seg = False
            seg += 1
        # terminator
        term, ta, tb = int(blk["term"]), str(int(blk["a"])), str(int(blk["b"]))
        if partner is not None:
            pb = self.dp.blocks[partner]
            if int(pb["a"]) != int(blk["a"]):
                ta = f"(sB_ ? {int(pb['a'])} : {ta})"
            if int(pb["b"]) != int(blk["b"]):
                tb = f"(sB_ ? {int(pb['b'])} : {tb})"
        body.append("  if (!ok) return false;")
        if self.cached_vars:
            body.insert(decl_at, "  uint64_t " + ", ".join(f"r{v} = 0" for v in sorted(self.cached_vars)) + ";")
        if all_sp:
            body.insert(decl_at, "  int " + ", ".join(f"sp{r} = 0" for r in sorted(all_sp)) + ";")
        if term == 1:
            c = int(blk["cond"])
            cv = f"s{c}" if c in locals_ else f"{self.ptr(c)}[0]"
            body.append(f"  const bool cond_ = {cv} != 0;")
        else:
            body.append("  const bool cond_ = false;")
        body.append(f"  return finish_block(a, ln, {term}, {ta}, {tb}, cond_, {int(blk['op_count']) + 1}, f, pc_, psp_);")
        body.append("}")
        return "\n".join(body)

    def emit(self) -> str:
        n = len(self.dp.blocks)
        out = ["// generated by paper_1910_11141_b200/codegen.py — do not edit",
               f"// options: {sorted(OPT.items())}", "#pragma once",
               f"#define LSB_GEN_STAGED {int(self.opt['staged'])}",
               f"#define LSB_GEN_OOL {int(self.opt['ool'])}",
               '#include "lsb_gen_rt.cuh"', "namespace lsbgen {",
               "// The current pc and pc-stack pointer live in registers (the engine writes them",
               "// back when a launch ends); memory keeps only the return addresses below the top.",
               "__device__ __forceinline__ bool finish_block(const VMArgs& a, const Lane& ln, int term, int ta, int tb,",
               "                                             bool cond, int pos, StepFault& f, int& pc, int& psp) {",
               "  switch (term) {",
               "    case LS_JUMP: pc = ta; return false;",
               "    case LS_BRANCH: pc = cond ? ta : tb; return false;",
               "    case LS_PUSHJUMP:",
               "      ln.pcs[(psp - 1) * ln.L + ln.t] = tb;",
               "      if (psp >= a.depth + 1) { pc = tb; f = StepFault{pos, LS_RUN_OVERFLOW, -1, 0}; return false; }",
               "      ++psp; pc = ta; return false;",
               "    default:",
               "      if (psp < 1) { f = StepFault{pos, LS_RUN_UNDERFLOW, -1, 0}; return false; }",
               "      --psp;",
               "      if (psp < 1) return false;",
               "      pc = ln.pcs[(psp - 1) * ln.L + ln.t];",
               "      return pc == a.halt;",
               "  }",
               "}"]
        pairs = self.find_pairs()
        for b in range(n):
            if b in pairs and pairs[b] < b:
                continue  # generated with its partner
            out.append(self.block(b, pairs.get(b)))
        out.append("__device__ __forceinline__ bool gen_exec_block(const VMArgs& a, const Lane& ln, int b, bool active,")
        out.append("                                               long long chain, StepFault& f, double* sm,")
        out.append("                                               int& pc_, int& psp_) {")
        out.append("  switch (b) {")
        for b in range(n):
            fb = min(b, pairs[b]) if b in pairs else b
            out.append(f"    case {b}: return gb_{fb}(a, ln, active, chain, f, sm, pc_, psp_);")
        out.append("  }")
        out.append("  return false;")
        out.append("}")
        out.append("// the block whose lanes share a warp step with block b (identical code), or -1")
        out.append("__device__ __forceinline__ int gen_pair(int b) {")
        out.append("  switch (b) {")
        for b, pb in sorted(pairs.items()):
            out.append(f"    case {b}: return {pb};")
        out.append("  }")
        out.append("  return -1;")
        out.append("}")
        out.append("}  // namespace lsbgen")
        return "\n".join(out) + "\n"


def generate(dp: DeviceProgram) -> str:
    """CUDA source of the program-specialised block functions."""
    return _Gen(dp).emit()


def library_for(dp: DeviceProgram, *, build: bool = True, verbose: bool = False) -> Path | None:
    """Path of the specialised C-ABI library for `dp`; compiles it if missing and `build`."""
    src = generate(dp)
    h = hashlib.sha256((src + _build.source_digest()).encode()).hexdigest()[:16]
    lib = GEN_DIR / f"liblockstep_b200_{h}.so"
    if lib.exists():
        return lib
    if not build:
        return None
    GEN_DIR.mkdir(parents=True, exist_ok=True)
    hdr = GEN_DIR / f"gen_{h}.cuh"
    hdr.write_text(src)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [_build._nvcc(), *_build.NVCC_FLAGS, "-diag-suppress", "177,550", "-I", str(_build.ROOT / "include"), "-I", str(_build.CSRC),
           f"-DLSB_GENERATED=\"{hdr}\"", f"-DLSB_BPF={OPT['bpf']}", f"-DLSB_EW_UNROLL={OPT['ewu']}",
           f"-DLSB_SB_PROFILE={OPT['sbprof']}", f"-DLSB_BLOCK_PROFILE={OPT['bprof']}", f"-DLSB_WARPS_MAX={OPT['wmax']}", f"-DLSB_LF_KC={OPT['lfkc']}",
           f"-DLSB_SB_INLINE={OPT['sbinline']}", f"-DLSB_WG_INLINE={OPT['wginline']}", "-o", str(tmp), str(_build.CSRC / "engine.cu")]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=str(_build.ROOT))
    os.replace(tmp, lib)
    return lib
