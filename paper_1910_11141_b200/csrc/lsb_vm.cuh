// lsb_vm.cuh — device core of the B200 program-counter VM: machine layout,
// op execution, warp-cooperative target contractions, fused superblocks.
//
// Storage. Every group of L lanes owns a workspace of `group_rows` rows of L
// 8-byte words ("lane-minor": element i of a lane's vector lives at row
// base+i, column = lane), so one warp touching element i of 32 lanes issues a
// single coalesced 256-byte access. Non-stacked variables have fixed rows
// laid out by the lowering (temporaries share an arena; views alias rows);
// stacked variables own depth x width rows and a per-lane stack pointer, the
// top slot being the one under the pointer (reference runtime.py:442-512).
//
// Ops arrive "resolved" (ROp): the machine precomputes each operand's base
// row, stack-pointer row and width, so executing an op costs one descriptor
// read plus the data accesses — no per-operand table walks.
#pragma once
#include <cstdint>

#include "../../include/lockstep_b200.h"
#include "lsb_dmma.cuh"
#include "lsb_tc.cuh"
#include "lsb_ops.cuh"

#ifndef LSB_LF_KC
#define LSB_LF_KC 2  // n-tiles per superblock kick pass
#endif

namespace lsbvm {

using lsb::as_f64;
using lsb::f64_bits;

constexpr int kMaxTargets = 8;
constexpr int kMaxLanes = 1024;
constexpr unsigned kFull = 0xffffffffu;

struct DevTarget {
  int kind = 0, dim = 0, n = 0;
  const double* P = nullptr;   // gaussian: precision (d x d, row-major); logreg: sx (n x d)
  const double* PT = nullptr;  // transpose of the above
  double norm = 0.0;
  // DMMA B operands in fragment order (lsb_dmma.cuh)
  const double* B1 = nullptr;  // gaussian: P (d x d);   logreg: sx^T (d x n)
  int KS1 = 0, NT1 = 0;
  const double* B2 = nullptr;  // logreg: sx (n x d)
  int KS2 = 0, NT2 = 0;
};

// One op with its operands resolved against the machine's storage layout.
struct ROp {
  int opcode, action, nin, kind;
  int width;               // output width (words)
  int out;                 // output (or popped) variable id, for fault reports
  int out_row, out_sp;     // output base row; stack-pointer row or -1
  int in_row[3], in_sp[3], in_w[3], in_kind[3];
  int imm0, imm1, imm2;
  int pad;                 // fused leaf logpdf row (superblock: written, LOGPDF: read) or -1
  long long bits;          // const payload; superblock: g_row | i_row << 32 (rows, -1 = none)
};

struct RBlock {
  int op_begin, op_count, term, a, b, grads;
  int cond_row, cond_sp, cond_w;
  int pad;
};

struct FaultRec {
  unsigned long long key;  // lowest wins
  int kind;                // LS_RUN_OVERFLOW / LS_RUN_UNDERFLOW
  int var;                 // -1 = pc stack
  int block;
  int detail;              // 1 = underflow of an update (write_top)
  long long chain;
};

struct VMArgs {
  const RBlock* blocks;
  const ROp* ops;
  int n_blocks, halt, entry;
  int n_inputs;
  const int* input_rows;        // slot-0 base row of each input var
  int output_row, output_sp, out_width;
  int n_sp_rows;                // stacked vars + 1 (pc)
  DevTarget targets[kMaxTargets];
  long long z;
  int depth;
  int lanes;                    // lanes per group
  int group_rows;
  uint64_t* ws;
  int* sp;                      // [groups][n_sp_rows][lanes]
  int* pcs;                     // [groups][depth+1][lanes]
  long long* chain_of;          // [groups][lanes]  (-1 free, -2 exhausted)
  const uint64_t* const* inputs;
  const int* input_width;
  uint64_t* output;             // [z][out_width]
  unsigned long long* next_chain;
  int refill, sched, exact_logpdf;
  long long max_steps;
  long long* group_steps;
  int* group_done;
  int* trace_block;
  int* trace_active;
  long long trace_cap;
  long long* trace_n;
  long long* blk_steps;
  long long* blk_active;
  long long* blk_cycles;        // [groups][n_blocks] SM clock cycles spent in each block
  unsigned long long* useful;
  unsigned long long* launched;
  int n_groups;
  int lf_smem_per_warp;
  // warp engine: one target's B fragments staged in shared memory at offset 0
  const double* stage_src;
  int stage_doubles;            // 0 = nothing staged
  int stage_target;
  int* lane_trace;
  int* lane_trace_len;
  int lane_trace_cap;
  int* gtrace;                  // warp engine: [groups][gtrace_cap] block | active << 16
  int* gtrace_len;              // [groups] records written (may exceed the cap)
  int gtrace_cap;
  FaultRec* fault;              // [n_groups] one fault slot per group
  int* abort_flag;
  int* paused;
  const unsigned* bkey;         // [n_blocks] schedule key of each block (block index in bits 0..15)
  // fp32 arm: the warps of a warpgroup meet at tensor-core superblocks (lsb_tc_leapfrog.cuh)
  int wg;
  // fp32 arm (lsb_tc_leapfrog.cuh): leapfrog superblocks on tcgen05 (3xTF32), the target's
  // precision matrix as a K-major TF32 hi/lo image staged in shared memory at byte offset
  // tc_smem_off by one bulk copy; nullptr = fp64 (DMMA) superblocks
  const void* tc_img;
  int tc_img_bytes, tc_half_bytes, tc_lbo, tc_sbo, tc_smem_off;
};

// Schedule key of a live lane at block `pc` with pc-stack depth `psp` (keyed rules pick the
// least): min_pc keys are the block index; priority keys rank blocks (host: pc_vm.block_keys);
// the local rule (paper Alg. 1, reference local_exec.py) runs the deepest activation first.
__device__ __forceinline__ unsigned lane_key(const VMArgs& a, int pc, int psp) {
  const unsigned k = __ldg(&a.bkey[pc]);
  if (a.sched != LS_SCHED_LOCAL) return k;
  const unsigned d = psp < 0 ? 0u : (psp > 255 ? 255u : (unsigned)psp);
  return ((255u - d) << 24) | (k & 0x00ffffffu);
}

struct Lane {
  uint64_t* ws;  // group workspace
  int* sp;       // group stack pointers
  int* pcs;      // group pc stack
  int t, L;

  __device__ __forceinline__ uint64_t* row(int r) const { return ws + (size_t)r * L + t; }
  __device__ __forceinline__ int& sp_row(int s) const { return sp[s * L + t]; }
  // current top of a variable given its base row / sp row / width
  __device__ __forceinline__ uint64_t* top(int base, int s, int w) const {
    if (s >= 0) {
      int p = sp_row(s) - 1;
      base += (p < 0 ? 0 : p) * w;
    }
    return row(base);
  }
  __device__ __forceinline__ const uint64_t* in(const ROp& op, int j) const {
    return top(op.in_row[j], op.in_sp[j], op.in_w[j]);
  }
};

__device__ __forceinline__ int64_t as_i64_any(uint64_t w, int kind) {
  return kind == LS_F64 ? lsb::f64_to_i64(as_f64(w)) : (int64_t)w;
}

// The fused draw_normals function (LS_OP_NORMALS): the exact op sequence of the
// NUTS-lite source (reference workloads.py draw_normals), one loop instead of
// 13 ops per normal — z_a = sqrt(0 - 2 log(1 - u_a)) cos(2 pi u_b), z_b = .. sin ..,
// u_j = rng_uniform(key, c + j); then c + 2 * pairs.
__device__ __forceinline__ void normals_lane(uint64_t* dst, int stride, int64_t key, double c, int k, int pairs) {
  constexpr double kTwoPi = 6.283185307179586;
#pragma unroll 1
  for (int pr = 0; pr < pairs; ++pr) {
    const int ia = 2 * pr, ib = 2 * pr + 1;
    const double ua = lsb::rng_uniform(key, lsb::f64_to_i64(__dadd_rn(c, (double)ia)));
    const double ub = lsb::rng_uniform(key, lsb::f64_to_i64(__dadd_rn(c, (double)ib)));
    const double r = __dsqrt_rn(__dsub_rn(0.0, __dmul_rn(2.0, log(__dsub_rn(1.0, ua)))));
    dst[(size_t)ia * stride] = f64_bits(__dmul_rn(r, cos(__dmul_rn(kTwoPi, ub))));
    if (ib < k) dst[(size_t)ib * stride] = f64_bits(__dmul_rn(r, sin(__dmul_rn(kTwoPi, ub))));
  }
  dst[(size_t)k * stride] = f64_bits(__dadd_rn(c, (double)(2 * pairs)));
}

// ---- per-lane target densities (reference workloads.py:186-228) --------------------

struct LrMargin {  // p(i) = logaddexp(0, -m_i) with m_i = w . sx_i
  const uint64_t* w;
  int stride, d;
  const double* sx;
  __device__ double operator()(int i) const {
    const double* r = sx + (size_t)i * d;
    double m = 0.0;
    for (int j = 0; j < d; ++j) m = fma(as_f64(w[(size_t)j * stride]), __ldg(r + j), m);
    return lsb::np_logaddexp(0.0, -m);
  }
};

__device__ inline double target_logpdf(const DevTarget& tg, const uint64_t* x, int stride, int exact) {
  if (tg.kind == LS_TARGET_GAUSSIAN) {
    if (exact) return lsb::gauss_logpdf_exact(x, stride, tg.dim, tg.P, tg.norm);
    double acc = 0.0;
    for (int j = 0; j < tg.dim; ++j) {
      const double* col = tg.PT + (size_t)j * tg.dim;
      double px = 0.0;
      for (int i = 0; i < tg.dim; ++i) px = fma(as_f64(x[(size_t)i * stride]), __ldg(col + i), px);
      acc = fma(as_f64(x[(size_t)j * stride]), px, acc);
    }
    return tg.norm - 0.5 * acc;
  }
  const double lik = lsb::pairwise(LrMargin{x, stride, tg.dim, tg.P}, 0, tg.n);
  const double ww = lsb::dot_lane(x, x, tg.dim, stride);
  return __dsub_rn(-__dadd_rn(0.0, lik), __dmul_rn(0.5, ww));
}

__device__ inline void target_grad(const DevTarget& tg, const uint64_t* x, int stride, uint64_t* out) {
  const int d = tg.dim;
  if (tg.kind == LS_TARGET_GAUSSIAN) {
    for (int j = 0; j < d; ++j) {
      const double* col = tg.PT + (size_t)j * d;
      double acc = 0.0;
      for (int i = 0; i < d; ++i) acc = fma(as_f64(x[(size_t)i * stride]), __ldg(col + i), acc);
      out[(size_t)j * stride] = f64_bits(-acc);
    }
    return;
  }
  for (int j = 0; j < d; ++j) out[(size_t)j * stride] = f64_bits(0.0);
  for (int i = 0; i < tg.n; ++i) {
    const double* r = tg.P + (size_t)i * d;
    double m = 0.0;
    for (int j = 0; j < d; ++j) m = fma(as_f64(x[(size_t)j * stride]), __ldg(r + j), m);
    const double s = lsb::lr_sig(m);
    for (int j = 0; j < d; ++j) {
      uint64_t* o = out + (size_t)j * stride;
      *o = f64_bits(fma(s, __ldg(r + j), as_f64(*o)));
    }
  }
  for (int j = 0; j < d; ++j) {
    uint64_t* o = out + (size_t)j * stride;
    *o = f64_bits(__dsub_rn(as_f64(*o), as_f64(x[(size_t)j * stride])));
  }
}

// Elementwise loop with 8 loads in flight before the stores (memory-level
// parallelism for the latency-bound copies that dominate NUTS-lite's packing).
// Loads-then-stores is safe when dst aliases an input element-for-element.
template <class F>
__device__ __forceinline__ void ew8(int w, uint64_t* dst, int L, const F& f) {
  int i = 0;
  for (; i + 8 <= w; i += 8) {
    uint64_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = f(i + j);
#pragma unroll
    for (int j = 0; j < 8; ++j) dst[(size_t)(i + j) * L] = v[j];
  }
  for (; i < w; ++i) dst[(size_t)i * L] = f(i);
}

// Computes op into dst for one lane. x, y, u: current tops of the inputs.
__device__ inline void compute_op(const VMArgs& a, const ROp& op, const uint64_t* x, const uint64_t* y,
                                  const uint64_t* u, uint64_t* dst, int L) {
  const int w = op.width;
  const bool f = op.kind == LS_F64;
#define X(i) x[(size_t)(i) * L]
#define Y(i) y[(size_t)(i) * L]
#define U(i) u[(size_t)(i) * L]
#define D(i) dst[(size_t)(i) * L]
  switch (op.opcode) {
    case LS_OP_CONST: D(0) = (uint64_t)op.bits; break;
    case LS_OP_ID: if (dst != x) ew8(w, dst, L, [&](int i) { return X(i); }); break;
    case LS_OP_ADD:
      if (f) ew8(w, dst, L, [&](int i) { return f64_bits(__dadd_rn(as_f64(X(i)), as_f64(Y(i)))); });
      else ew8(w, dst, L, [&](int i) { return X(i) + Y(i); });
      break;
    case LS_OP_SUB:
      if (f) ew8(w, dst, L, [&](int i) { return f64_bits(__dsub_rn(as_f64(X(i)), as_f64(Y(i)))); });
      else ew8(w, dst, L, [&](int i) { return X(i) - Y(i); });
      break;
    case LS_OP_MUL:
      if (f) ew8(w, dst, L, [&](int i) { return f64_bits(__dmul_rn(as_f64(X(i)), as_f64(Y(i)))); });
      else ew8(w, dst, L, [&](int i) { return (uint64_t)((unsigned long long)X(i) * (unsigned long long)Y(i)); });
      break;
    case LS_OP_DIV:
      ew8(w, dst, L, [&](int i) -> uint64_t {
        if (f) return f64_bits(__ddiv_rn(as_f64(X(i)), as_f64(Y(i))));
        const int64_t p = (int64_t)X(i), q = (int64_t)Y(i);  // numpy floor_divide, /0 -> 0
        if (q == 0) return 0;
        if (q == -1) return 0ull - (uint64_t)p;
        int64_t r = p / q;
        if ((p % q != 0) && ((p < 0) != (q < 0))) r -= 1;
        return (uint64_t)r;
      });
      break;
    case LS_OP_MIN:
    case LS_OP_MAX: {
      const bool mn = op.opcode == LS_OP_MIN;
      ew8(w, dst, L, [&](int i) -> uint64_t {
        if (f) {
          const double p = as_f64(X(i)), q = as_f64(Y(i));
          if (p != p) return f64_bits(p);
          if (q != q) return f64_bits(q);
          return f64_bits(mn ? (p <= q ? p : q) : (p >= q ? p : q));
        }
        const int64_t p = (int64_t)X(i), q = (int64_t)Y(i);
        return (uint64_t)(mn ? (p < q ? p : q) : (p > q ? p : q));
      });
      break;
    }
    case LS_OP_LE: D(0) = f ? (as_f64(X(0)) <= as_f64(Y(0))) : ((int64_t)X(0) <= (int64_t)Y(0)); break;
    case LS_OP_LT: D(0) = f ? (as_f64(X(0)) < as_f64(Y(0))) : ((int64_t)X(0) < (int64_t)Y(0)); break;
    case LS_OP_EQ: D(0) = f ? (as_f64(X(0)) == as_f64(Y(0))) : (X(0) == Y(0)); break;
    case LS_OP_AND: D(0) = (X(0) != 0) && (Y(0) != 0); break;
    case LS_OP_OR: D(0) = (X(0) != 0) || (Y(0) != 0); break;
    case LS_OP_NOT: D(0) = X(0) == 0; break;
    case LS_OP_NEG:
      ew8(w, dst, L, [&](int i) { return f ? f64_bits(-as_f64(X(i))) : (uint64_t)(0ull - X(i)); });
      break;
    case LS_OP_ABS:
      ew8(w, dst, L, [&](int i) -> uint64_t {
        if (f) return f64_bits(fabs(as_f64(X(i))));
        const int64_t p = (int64_t)X(i);
        return p < 0 ? (uint64_t)(0ull - (uint64_t)p) : (uint64_t)p;
      });
      break;
    case LS_OP_SQRT: ew8(w, dst, L, [&](int i) { return f64_bits(__dsqrt_rn(as_f64(X(i)))); }); break;
    case LS_OP_EXP: ew8(w, dst, L, [&](int i) { return f64_bits(exp(as_f64(X(i)))); }); break;
    case LS_OP_LOG: ew8(w, dst, L, [&](int i) { return f64_bits(log(as_f64(X(i)))); }); break;
    case LS_OP_SIN: ew8(w, dst, L, [&](int i) { return f64_bits(sin(as_f64(X(i)))); }); break;
    case LS_OP_COS: ew8(w, dst, L, [&](int i) { return f64_bits(cos(as_f64(X(i)))); }); break;
    case LS_OP_FLOOR: ew8(w, dst, L, [&](int i) { return f64_bits(floor(as_f64(X(i)))); }); break;
    case LS_OP_SELECT: {
      const uint64_t* src = X(0) != 0 ? y : u;
      if (src != dst) ew8(w, dst, L, [&](int i) { return src[(size_t)i * L]; });
      break;
    }
    case LS_OP_DOT: D(0) = f64_bits(lsb::dot_lane(x, y, op.in_w[0], L)); break;
    case LS_OP_AXPY: {
      const double s = as_f64(X(0));
      ew8(w, dst, L, [&](int i) { return f64_bits(__dadd_rn(__dmul_rn(s, as_f64(Y(i))), as_f64(U(i)))); });
      break;
    }
    case LS_OP_VGET: {
      const int vw = op.in_w[0];
      int64_t k = as_i64_any(Y(0), op.in_kind[1]);
      k = k < 0 ? 0 : (k > vw - 1 ? vw - 1 : k);
      D(0) = X(k);
      break;
    }
    case LS_OP_VSTORE: {
      int64_t k = as_i64_any(Y(0), op.in_kind[1]);
      k = k < 0 ? 0 : (k > w - 1 ? w - 1 : k);
      const uint64_t val = U(0);
      if (dst != x) ew8(w, dst, L, [&](int i) { return X(i); });
      D(k) = val;
      break;
    }
    case LS_OP_VCAT: {
      const int wa = op.in_w[0];
      if (dst != x) ew8(wa, dst, L, [&](int i) { return X(i); });
      ew8(w - wa, dst + (size_t)wa * L, L, [&](int i) { return Y(i); });
      break;
    }
    case LS_OP_VFILL: {
      const uint64_t v = X(0);
      ew8(w, dst, L, [&](int) { return v; });
      break;
    }
    case LS_OP_VSLICE:
      if (dst != x + (size_t)op.imm0 * L) ew8(w, dst, L, [&](int i) { return X(op.imm0 + i); });
      break;
    case LS_OP_RNG: {
      const int64_t k = as_i64_any(X(0), op.in_kind[0]);
      const int64_t c = as_i64_any(Y(0), op.in_kind[1]);
      D(0) = f64_bits(lsb::rng_uniform(k, c));
      break;
    }
    case LS_OP_NORMALS:
      normals_lane(dst, L, as_i64_any(X(0), op.in_kind[0]), as_f64(Y(0)), op.imm0, op.imm1);
      break;
    case LS_OP_LOGPDF: D(0) = f64_bits(target_logpdf(a.targets[op.imm0], x, L, a.exact_logpdf)); break;
    case LS_OP_GRAD: target_grad(a.targets[op.imm0], x, L, dst); break;
    default: break;
  }
#undef X
#undef Y
#undef U
#undef D
}

__device__ inline void write_output(const VMArgs& a, const Lane& ln, long long chain) {
  const uint64_t* src = ln.top(a.output_row, a.output_sp, a.out_width);
  uint64_t* dst = a.output + (size_t)chain * a.out_width;
  const int w = a.out_width;
  int i = 0;
  for (; i + 16 <= w; i += 16) {  // 16 loads in flight before the stores
    uint64_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = src[(size_t)(i + j) * ln.L];
#pragma unroll
    for (int j = 0; j < 16; ++j) dst[i + j] = v[j];
  }
  for (; i < w; ++i) dst[i] = src[(size_t)i * ln.L];
}

// Warp engine: the lanes in `hmask` halted this step; the whole warp writes each one's
// output row (thread t takes words t, t+32, ...), so every store instruction is one
// contiguous 256-byte run — which also makes a page-locked host destination
// (ls_machine_set_output_host) cheap to write across PCIe while the kernel runs.
__device__ __forceinline__ void warp_write_outputs(const VMArgs& a, const Lane& ln, unsigned hmask,
                                                   long long chain) {
  const int lane = threadIdx.x & 31;
  const uint64_t* mysrc = ln.top(a.output_row, a.output_sp, a.out_width);
  const int w = a.out_width;
  while (hmask) {
    const int l = __ffs(hmask) - 1;
    hmask &= hmask - 1;
    const uint64_t* src = (const uint64_t*)__shfl_sync(kFull, (unsigned long long)mysrc, l);
    const long long c = __shfl_sync(kFull, chain, l);
    uint64_t* dst = a.output + (size_t)c * w;
    for (int i0 = 0; i0 < w; i0 += 32 * 8) {
      uint64_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + 32 * j + lane;
        if (i < w) v[j] = src[(size_t)i * ln.L];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + 32 * j + lane;
        if (i < w) dst[i] = v[j];
      }
    }
  }
}

__device__ inline void init_lane(const VMArgs& a, const Lane& ln, long long chain) {
  // data stacks hold one live slot from the start (reference pc_vm.py:180-181)
  for (int r = 0; r + 1 < a.n_sp_rows; ++r) ln.sp_row(r) = 1;
  for (int k = 0; k < a.n_inputs; ++k) {
    const int w = a.input_width[k];
    const uint64_t* src = a.inputs[k] + (size_t)chain * w;
    uint64_t* dst = ln.row(a.input_rows[k]);
    for (int i = 0; i < w; ++i) dst[(size_t)i * ln.L] = src[i];
  }
  // pc stack seeded [halt, entry], pointer 2 (reference pc_vm.py:199-203)
  ln.pcs[0 * ln.L + ln.t] = a.halt;
  ln.pcs[1 * ln.L + ln.t] = a.entry;
  ln.sp_row(a.n_sp_rows - 1) = 2;
}

__device__ __forceinline__ void lane_trace_put(const VMArgs& a, long long chain, int block) {
  const int n = a.lane_trace_len[chain];
  if (n < a.lane_trace_cap) a.lane_trace[(size_t)chain * a.lane_trace_cap + n] = block;
  a.lane_trace_len[chain] = n + 1;
}

// ---- warp-cooperative contractions (DMMA) ------------------------------------------------

// row g (0..7) of m-tile mt: the (8*mt+g)-th participating lane, or -1
__device__ __forceinline__ int mtile_lane(unsigned mask, int n, int mt, int g) {
  const int idx = 8 * mt + g;
  return idx < n ? (int)__fns(mask, 0, idx + 1) : -1;
}

// n-tiles (of 8 columns) up to which a target counts as narrow: the register-momentum
// superblock and single-m-tile contractions; wider targets take warp_gauss_wide
constexpr int kLfRegMaxTiles = 16;

// The CTA's shared-memory copy of target `t`'s B fragments, or nullptr (warp engine).
__device__ __forceinline__ const double* staged_B(const VMArgs& a, int t) {
  extern __shared__ double lsb_dyn_smem[];
  return (a.stage_doubles > 0 && t == a.stage_target) ? lsb_dyn_smem : nullptr;
}

// The fast gaussian logpdf from the contraction quad = q.(P q) (shared by
// warp_gauss and the superblock's fused leaf logpdf, so both round identically).
__device__ __forceinline__ double gauss_lp_from_quad(double norm, double quad) {
  return __dsub_rn(norm, __dmul_rn(0.5, quad));
}

// Shared-memory row stride (doubles) of a staged 8-chain tile: DMMA A-fragment
// loads (8 rows x 4 cols, 64-bit) are bank-conflict free.
__host__ __device__ __forceinline__ int lf_stride_q(int d) { int s = (d + 7) / 8 * 8; return s + ((12 - s % 16) + 16) % 16; }

// Stage x[0..d) of m-tile mt's 8 chains (rows; zero padded to SQ columns and for
// missing chains) into Xs[8][SQ]. Thread (k % 4, row r) reads x[k][lane_r], so each
// load instruction covers 4 workspace rows x 8 lanes (64-byte runs when the lanes
// are contiguous), 8 loads in flight per thread.
// kBatch loads in flight per thread; the superblock passes its whole tile (one round trip).
template <int kBatch = 8>
__device__ __forceinline__ void stage_mtile(double* Xs, int SQ, const uint64_t* myx, unsigned mask, int n,
                                            int mt, int d) {
  const int lane = threadIdx.x & 31;
  const int r = lane & 7, kq = lane >> 3;
  const int lr = mtile_lane(mask, n, mt, r);
  const uint64_t* xg = (const uint64_t*)__shfl_sync(kFull, (unsigned long long)myx, lr < 0 ? 0 : lr);
  for (int k0 = 0; k0 < SQ; k0 += 4 * kBatch) {
    double v[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int k = k0 + 4 * i + kq;
      v[i] = (lr >= 0 && k < d) ? as_f64(xg[(size_t)k * 32]) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int k = k0 + 4 * i + kq;
      if (k < SQ) Xs[r * SQ + k] = v[i];
    }
  }
}

template <bool SB, bool SX>
__device__ inline void warp_gauss_impl(const DevTarget& tg, const double* Bf, bool part, const uint64_t* xp,
                                       uint64_t* dst, bool want_logpdf, double* Xs);

// Wide gaussian targets (d > 128, e.g. BASELINE config 5 at d = 1000): the precision
// matrix (8 MB at d = 1000) does not fit on chip, so every B fragment read from L2 feeds
// all of the warp's m-tiles (up to 4 x 8 chains) and every A fragment 4 n-tiles: 8 DMMAs
// per 6 fragment loads instead of 1 per 2. Accumulation order per output element and the
// logpdf's fma order are warp_gauss_impl's, so results are bit-identical.
__device__ __noinline__ void warp_gauss_wide(const DevTarget& tg, bool part, const uint64_t* xp, uint64_t* dst,
                                             bool want_logpdf) {
  constexpr int NTC = 4;
  const int lane = threadIdx.x & 31, g = lane >> 2;
  const unsigned mask = __ballot_sync(kFull, part);
  const int n = __popc(mask);
  if (n == 0) return;
  const int MT = (n + 7) / 8;
  const int d = tg.dim, KS = tg.KS1, NT = tg.NT1;
  const uint64_t* xg[4];
  uint64_t* dg[4];
  bool okr[4];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int src = mt < MT ? mtile_lane(mask, n, mt, g) : -1;
    okr[mt] = src >= 0;
    xg[mt] = (const uint64_t*)__shfl_sync(kFull, (unsigned long long)xp, src < 0 ? 0 : src);
    dg[mt] = (uint64_t*)__shfl_sync(kFull, (unsigned long long)dst, src < 0 ? 0 : src);
  }
  double quad[4] = {0.0, 0.0, 0.0, 0.0};
  for (int nt0 = 0; nt0 < NT; nt0 += NTC) {
    const int ntc = min(NTC, NT - nt0);
    double acc[4][NTC][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int j = 0; j < NTC; ++j) acc[mt][j][0] = acc[mt][j][1] = 0.0;
    const double* bp = tg.B1 + (size_t)nt0 * 32 + lane;
    const size_t kstride = (size_t)NT * 32;
#pragma unroll 1
    for (int ks = 0; ks < KS; ++ks) {
      const int k = 4 * ks + (lane & 3);
      double av[4], bv[NTC];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) av[mt] = (okr[mt] && k < d) ? as_f64(xg[mt][(size_t)k * 32]) : 0.0;
#pragma unroll
      for (int j = 0; j < NTC; ++j) bv[j] = j < ntc ? lsb::ldg_keep(bp + j * 32) : 0.0;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
        if (mt < MT) {  // warp-uniform
#pragma unroll
          for (int j = 0; j < NTC; ++j) lsb::dmma(acc[mt][j], av[mt], bv[j]);
        }
      bp += kstride;
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      if (!okr[mt]) continue;
#pragma unroll
      for (int j = 0; j < NTC; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * (nt0 + j) + 2 * (lane & 3) + e;
          if (j < ntc && col < d) {
            if (want_logpdf) quad[mt] = fma(as_f64(xg[mt][(size_t)col * 32]), acc[mt][j][e], quad[mt]);
            else dg[mt][(size_t)col * 32] = f64_bits(-acc[mt][j][e]);
          }
        }
    }
  }
  if (want_logpdf) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      double q = quad[mt];
      q += __shfl_xor_sync(kFull, q, 1);
      q += __shfl_xor_sync(kFull, q, 2);
      if (okr[mt] && (lane & 3) == 0) dg[mt][0] = f64_bits(gauss_lp_from_quad(tg.norm, q));
    }
  }
}

// grad, or fast logpdf, of a gaussian target for every participating lane of the
// warp (lane-minor storage, stride 32). xp/dst: this lane's input and output.
// Bs: the staged B fragments (staged_B) or nullptr. sm/sm_doubles: the warp's
// shared-memory scratch; when it holds an 8-chain tile of x, the A operand is
// staged there (coalesced) instead of read from the workspace per k-step.
#ifndef LSB_WG_INLINE
#define LSB_WG_INLINE 0
#endif
#if LSB_WG_INLINE
__device__ __forceinline__
#else
__device__ inline
#endif
void warp_gauss(const DevTarget& tg, const double* Bs, bool part, const uint64_t* xp,
                                  uint64_t* dst, bool want_logpdf, double* sm, int sm_doubles) {
  if (tg.NT1 > kLfRegMaxTiles && Bs == nullptr) {
    warp_gauss_wide(tg, part, xp, dst, want_logpdf);
    return;
  }
  const bool sx = sm != nullptr && 8 * lf_stride_q(tg.dim) <= sm_doubles;
  if (Bs) {
    if (sx) warp_gauss_impl<true, true>(tg, Bs, part, xp, dst, want_logpdf, sm);
    else warp_gauss_impl<true, false>(tg, Bs, part, xp, dst, want_logpdf, nullptr);
  } else {
    if (sx) warp_gauss_impl<false, true>(tg, tg.B1, part, xp, dst, want_logpdf, sm);
    else warp_gauss_impl<false, false>(tg, tg.B1, part, xp, dst, want_logpdf, nullptr);
  }
}

template <bool SB, bool SX>
__device__ inline void warp_gauss_impl(const DevTarget& tg, const double* Bf, bool part, const uint64_t* xp,
                                       uint64_t* dst, bool want_logpdf, double* Xs) {
  const int lane = threadIdx.x & 31, g = lane >> 2;
  const unsigned mask = __ballot_sync(kFull, part);
  const int n = __popc(mask);
  const int d = tg.dim;
  const int SQ = lf_stride_q(d);
  for (int mt = 0; mt * 8 < n; ++mt) {
    const int src = mtile_lane(mask, n, mt, g);
    const uint64_t* xg = (const uint64_t*)__shfl_sync(kFull, (unsigned long long)xp, src < 0 ? 0 : src);
    uint64_t* dg = (uint64_t*)__shfl_sync(kFull, (unsigned long long)dst, src < 0 ? 0 : src);
    if constexpr (SX) {
      __syncwarp();
      stage_mtile(Xs, SQ, xp, mask, n, mt, d);
      __syncwarp();
    }
    auto x_at = [&](int k) -> double {
      if constexpr (SX) return Xs[g * SQ + k];
      else return (src >= 0 && k < d) ? as_f64(xg[(size_t)k * 32]) : 0.0;
    };
    double quad = 0.0;
    for (int nt0 = 0; nt0 < tg.NT1; nt0 += LSB_NT_CHUNK) {
      const int ntc = min(LSB_NT_CHUNK, tg.NT1 - nt0);
      LSB_NT_DISPATCH(ntc, {
        double acc[NTC][2];
        lsb::mtile_gemm<NTC, SB>(acc, Bf, tg.KS1, tg.NT1, nt0, x_at);
        _Pragma("unroll")
        for (int j = 0; j < NTC; ++j) {
          _Pragma("unroll")
          for (int e = 0; e < 2; ++e) {
            const int col = 8 * (nt0 + j) + 2 * (lane & 3) + e;
            if (src >= 0 && col < d) {
              if (want_logpdf) quad = fma(x_at(col), acc[j][e], quad);
              else dg[(size_t)col * 32] = f64_bits(-acc[j][e]);
            }
          }
        }
      });
    }
    if (want_logpdf) {
      quad += __shfl_xor_sync(kFull, quad, 1);
      quad += __shfl_xor_sync(kFull, quad, 2);
      if (src >= 0 && (lane & 3) == 0) dg[0] = f64_bits(gauss_lp_from_quad(tg.norm, quad));
    }
  }
  if constexpr (SX) __syncwarp();
}

// Logistic regression on the DMMA path for every participating lane, as one fused pass
// per 8-chain m-tile over blocks of 4 x 8 data points (reference workloads.py:216-228):
//   m = w sx^T (K = d, 4 independent n-tile accumulators, prefetched fragments) -> C frags
//   grad:   s = sigmoid(-m) (lr_sig);  G += s sx (K = data) <- s re-laid out as A fragments
//   logpdf: acc += logaddexp(0, -m) per thread, reduced over the row's 4 threads
// The margins never touch memory (FlashAttention-style fusion). w is staged as an 8-chain
// A tile in the warp's shared memory (stage_mtile); B1 = sx^T and B2 = sx are the target's
// fragment-ordered operands (L2-resident). NT2 = ceil(d/8) <= 16.
template <int NT2, bool LOGPDF, int NB>
__device__ __forceinline__ void lr_block(const DevTarget& tg, const double* Xs, int SQ, int nt0, double (&G)[NT2][2],
                                         double& lp) {
  const int lane = threadIdx.x & 31, g = lane >> 2;
  double acc[NB][2];
  lsb::mtile_gemm_pf<NB, false>(acc, tg.B1, tg.KS1, tg.NT1, nt0, [&](int k) -> double { return Xs[g * SQ + k]; });
  // thread (g, c = lane & 3) takes A2[g][k] for k = c of each GEMM2 k-step from the lane
  // holding s[g][k] in the C layout: lane 4g + k/2, element k & 1
  const int q0 = (lane & ~3) | ((lane & 3) >> 1), q1 = q0 + 2;
  const bool hi = (lane & 1) != 0;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int nt = nt0 + j;
    if (LOGPDF) {
      // padded data points (>= n) have zero margins: skip them
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (8 * nt + 2 * (lane & 3) + e < tg.n) lp = __dadd_rn(lp, lsb::np_logaddexp(0.0, -acc[j][e]));
      continue;
    }
    // padded data points have zero B1 columns and zero B2 rows: harmless
    const double s0 = lsb::lr_sig(acc[j][0]), s1 = lsb::lr_sig(acc[j][1]);
    const double u0 = __shfl_sync(kFull, s0, q0), u1 = __shfl_sync(kFull, s1, q0);
    const double v0 = __shfl_sync(kFull, s0, q1), v1 = __shfl_sync(kFull, s1, q1);
    const double a0 = hi ? u1 : u0, a1 = hi ? v1 : v0;
    const double* b0 = tg.B2 + (size_t)(2 * nt) * tg.NT2 * 32 + lane;
    if (2 * nt < tg.KS2) {
#pragma unroll
      for (int k = 0; k < NT2; ++k) lsb::dmma(G[k], a0, lsb::ldg_keep(b0 + k * 32));
    }
    if (2 * nt + 1 < tg.KS2) {
      const double* b1 = b0 + (size_t)tg.NT2 * 32;
#pragma unroll
      for (int k = 0; k < NT2; ++k) lsb::dmma(G[k], a1, lsb::ldg_keep(b1 + k * 32));
    }
  }
}

template <int NT2, bool LOGPDF>
__device__ void warp_lr_nt(const DevTarget& tg, bool part, const uint64_t* xp, uint64_t* dst, double* Xs) {
  const int lane = threadIdx.x & 31, g = lane >> 2;
  const unsigned mask = __ballot_sync(kFull, part);
  const int n = __popc(mask);
  const int d = tg.dim;
  const int SQ = lf_stride_q(d);
  for (int mt = 0; mt * 8 < n; ++mt) {
    const int src = mtile_lane(mask, n, mt, g);
    uint64_t* dg = (uint64_t*)__shfl_sync(kFull, (unsigned long long)dst, src < 0 ? 0 : src);
    __syncwarp();
    stage_mtile(Xs, SQ, xp, mask, n, mt, d);
    __syncwarp();
    double G[NT2][2];
#pragma unroll
    for (int j = 0; j < NT2; ++j) G[j][0] = G[j][1] = 0.0;
    double lp = 0.0;
    int nt0 = 0;
    for (; nt0 + 4 <= tg.NT1; nt0 += 4) lr_block<NT2, LOGPDF, 4>(tg, Xs, SQ, nt0, G, lp);
    switch (tg.NT1 - nt0) {
      case 3: lr_block<NT2, LOGPDF, 3>(tg, Xs, SQ, nt0, G, lp); break;
      case 2: lr_block<NT2, LOGPDF, 2>(tg, Xs, SQ, nt0, G, lp); break;
      case 1: lr_block<NT2, LOGPDF, 1>(tg, Xs, SQ, nt0, G, lp); break;
      default: break;
    }
    if (LOGPDF) {
      lp = __dadd_rn(lp, __shfl_xor_sync(kFull, lp, 1));
      lp = __dadd_rn(lp, __shfl_xor_sync(kFull, lp, 2));
      if (src >= 0 && (lane & 3) == 0) {
        const double ww = lsb::pairwise([&](int k) { return __dmul_rn(Xs[g * SQ + k], Xs[g * SQ + k]); }, 0, d);
        dg[0] = f64_bits(__dsub_rn(-lp, __dmul_rn(0.5, __dadd_rn(0.0, ww))));
      }
    } else if (src >= 0) {
#pragma unroll
      for (int j = 0; j < NT2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * j + 2 * (lane & 3) + e;
          if (col < d) dg[(size_t)col * 32] = f64_bits(__dsub_rn(G[j][e], Xs[g * SQ + col]));
        }
    }
    __syncwarp();
  }
}

// Logistic regression with the design streamed (every design of at least kLrStreamMinN
// points, e.g. BASELINE config 3 at 1000 x 25 and config 4 at 100k x 100 = 80 MB): reading
// sx fragment by fragment from L2 leaves one warp waiting on a load chain per 8 points.
// Instead sx streams through a per-warp shared-memory ring: lane 0 issues bulk async copies
// (cp.async.bulk, the TMA engine; completion counted in bytes on an mbarrier per stage) of
// kLrChunk contiguous data points, the next chunk in flight while one is consumed, and every
// chunk feeds BOTH GEMMs of the m-tile pass straight from shared memory — margins (B = sx^T:
// thread (g, c) reads point g, coordinate 4ks + c) and G += s sx (B = sx: point 4kk + c,
// coordinate 8j + g) — so sx is read once per m-tile pass instead of twice in two fragment
// orders. DMMA results land ~100 cycles after issue, so a chunk's margins accumulate in
// eight independent chains (four n-tiles x even / odd k-steps) and its 13 gradient
// accumulators interleave; the sigmoid is branch-free (no divergence between lanes).
// Per-warp shared memory: the w tile, the ring, the barriers.
constexpr int kLrStreamMinN = 512;  // designs at least this tall stream (host: engine.cu)
constexpr int kLrChunk = 32;        // data points per stage (four 8-point n-tiles)
constexpr int kLrStages = 2;        // one chunk in flight while one is consumed (copy << compute)
constexpr int kLrNt = kLrChunk / 8;
__host__ __device__ __forceinline__ int lr_stream_doubles(int d) {
  return 8 * lf_stride_q(d) + kLrStages * kLrChunk * d + kLrStages;  // + barriers (even)
}

// The body is force-inlined where the program-specialised code calls it for its target's
// NT2 (measured: as an out-of-line call inside the VM kernel the G accumulators spill and a
// chunk takes twice as long as the same code compiled on its own); the interpreter calls
// the out-of-line warp_lr_stream below.
#ifdef LSB_GENERATED
#define LSB_LRS_NAME warp_lr_stream_body
#define LSB_LRS_QUAL __forceinline__
#else  // the interpreter library: the body itself is the out-of-line warp_lr_stream (the same
       // text as a wrapper around a force-inlined body made ptxas run for over an hour)
#define LSB_LRS_NAME warp_lr_stream
#define LSB_LRS_QUAL __noinline__
#endif
template <int NT2, bool LOGPDF>
__device__ LSB_LRS_QUAL void LSB_LRS_NAME(const DevTarget& tgr, bool part, const uint64_t* xp, uint64_t* dst,
                                          double* sm) {
  const int lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  const unsigned mask = __ballot_sync(kFull, part);
  const int n_act = __popc(mask);
  if (n_act == 0) return;
  const int d = tgr.dim, n = tgr.n, SQ = lf_stride_q(d), KS = (d + 3) / 4;
  const double* const sx = tgr.P;
  double* Xs = sm;
  double* ring = sm + 8 * SQ;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kLrStages * kLrChunk * d);
  const int MT = (n_act + 7) / 8, nch = (n + kLrChunk - 1) / kLrChunk, total = MT * nch;
  if (lane == 0) {
    for (int s = 0; s < kLrStages; ++s) lsbtc::mbar_init(&bars[s], 1);
    lsbtc::fence_barrier_init();
  }
  __syncwarp();
  // lane 0: chunk ch into stage st. The stage's previous contents were consumed (into
  // registers) by every lane before the __syncwarp that precedes the issue.
  auto issue = [&](int ch, int st) {
    const int pts = min(kLrChunk, n - ch * kLrChunk);
    const uint32_t bytes = (uint32_t)(pts * d * 8) & ~15u;  // an odd tail word: plain load below
    lsbtc::mbar_expect_tx(&bars[st], bytes);
    if (bytes) lsbtc::bulk_g2s(ring + (size_t)st * kLrChunk * d, sx + (size_t)ch * kLrChunk * d, bytes, &bars[st]);
  };
  // the item sequence (m-tile pass mt, chunk ch) is walked twice: issue runs kLrStages ahead
  int ich = 0, ist = 0;
  const int pre = min(kLrStages, total);
  if (lane == 0)
    for (int i = 0; i < pre; ++i) {
      issue(ich, ist);
      if (++ich == nch) ich = 0;
      if (++ist == kLrStages) ist = 0;
    }
  const int q0 = (lane & ~3) | (c >> 1), q1 = q0 + 2;
  const bool hi = (lane & 1) != 0;
  double G[NT2][2];
  double lp = 0.0;
  int src = -1;
  int mt = 0, ch = 0, st = 0;
  uint32_t par = 0;
  for (int it = 0; it < total; ++it) {
    if (ch == 0) {  // a new m-tile pass: stage its 8 chains' w, clear the accumulators
      src = mtile_lane(mask, n_act, mt, g);
      __syncwarp();
      stage_mtile(Xs, SQ, xp, mask, n_act, mt, d);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < NT2; ++j) G[j][0] = G[j][1] = 0.0;
      lp = 0.0;
    }
    const int p0 = ch * kLrChunk, pts = min(kLrChunk, n - p0);
    const double* X = ring + (size_t)st * kLrChunk * d;
    lsbtc::mbar_wait(&bars[st], par);
    if (((pts * d) & 1) && lane == 0) {
      const size_t last = (size_t)pts * d - 1;
      const_cast<double*>(X)[last] = __ldg(sx + (size_t)p0 * d + last);
    }
    __syncwarp();
    // margins of the chunk's 32 points (four n-tiles) for the m-tile's 8 chains, C layout,
    // as eight independent DMMA chains (n-tile x even / odd k-step); rows past the chunk's
    // points read as zero
    double acc[kLrNt][2][2] = {};
    {
      const double* b0 = X + (size_t)g * d + c;
#pragma unroll 2
      for (int ks = 0; ks < KS; ks += 2) {
        const int k = 4 * ks + c, k2 = k + 4;
        const double a0 = Xs[g * SQ + k], a1 = Xs[g * SQ + k2];  // zero padded to SQ >= 4 KS + 4
        const bool in0 = k < d, in1 = k2 < d;
#pragma unroll
        for (int t = 0; t < kLrNt; ++t) {
          const bool pr = 8 * t + g < pts;
          lsb::dmma(acc[t][0], a0, (pr && in0) ? b0[(size_t)8 * t * d + 4 * ks] : 0.0);
          lsb::dmma(acc[t][1], a1, (pr && in1) ? b0[(size_t)8 * t * d + 4 * ks + 4] : 0.0);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kLrNt; ++t) {
      const double m0 = __dadd_rn(acc[t][0][0], acc[t][1][0]), m1 = __dadd_rn(acc[t][0][1], acc[t][1][1]);
      if (LOGPDF) {
        if (8 * t + 2 * c < pts) lp = __dadd_rn(lp, lsb::np_logaddexp(0.0, -m0));
        if (8 * t + 2 * c + 1 < pts) lp = __dadd_rn(lp, lsb::np_logaddexp(0.0, -m1));
        continue;
      }
      const double s0 = 8 * t + 2 * c < pts ? lsb::lr_sig_nb(m0) : 0.0;
      const double s1 = 8 * t + 2 * c + 1 < pts ? lsb::lr_sig_nb(m1) : 0.0;
      const double u0 = __shfl_sync(kFull, s0, q0), u1 = __shfl_sync(kFull, s1, q0);
      const double v0 = __shfl_sync(kFull, s0, q1), v1 = __shfl_sync(kFull, s1, q1);
      const double a0 = hi ? u1 : u0, a1 = hi ? v1 : v0;
      const bool r0 = 8 * t + c < pts, r1 = 8 * t + 4 + c < pts;
      const double* b0 = X + (size_t)(8 * t + c) * d + g;
      const double* b1 = b0 + (size_t)4 * d;
#pragma unroll
      for (int j = 0; j < NT2; ++j) {
        const bool col = 8 * j + g < d;
        lsb::dmma(G[j], a0, (r0 && col) ? b0[8 * j] : 0.0);
        lsb::dmma(G[j], a1, (r1 && col) ? b1[8 * j] : 0.0);
      }
    }
    __syncwarp();  // every lane is done with the stage before it is refilled
    if (lane == 0 && it + kLrStages < total) {
      issue(ich, ist);
      if (++ich == nch) ich = 0;
      if (++ist == kLrStages) ist = 0;
    }
    if (ch == nch - 1) {  // the m-tile pass is complete
      uint64_t* dg = (uint64_t*)__shfl_sync(kFull, (unsigned long long)dst, src < 0 ? 0 : src);
      if (LOGPDF) {
        lp = __dadd_rn(lp, __shfl_xor_sync(kFull, lp, 1));
        lp = __dadd_rn(lp, __shfl_xor_sync(kFull, lp, 2));
        if (src >= 0 && c == 0) {
          const double ww = lsb::pairwise([&](int k) { return __dmul_rn(Xs[g * SQ + k], Xs[g * SQ + k]); }, 0, d);
          dg[0] = f64_bits(__dsub_rn(-lp, __dmul_rn(0.5, __dadd_rn(0.0, ww))));
        }
      } else if (src >= 0) {
#pragma unroll
        for (int j = 0; j < NT2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 8 * j + 2 * c + e;
            if (col < d) dg[(size_t)col * 32] = f64_bits(__dsub_rn(G[j][e], Xs[g * SQ + col]));
          }
      }
    }
    if (++st == kLrStages) {
      st = 0;
      par ^= 1u;
    }
    if (++ch == nch) {
      ch = 0;
      ++mt;
    }
  }
  __syncwarp();
  if (lane == 0)
    for (int s = 0; s < kLrStages; ++s)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(lsbtc::smem_u32(&bars[s])) : "memory");
  __syncwarp();
}

#ifdef LSB_GENERATED
template <int NT2, bool LOGPDF>
__device__ __noinline__ void warp_lr_stream(const DevTarget& tg, bool part, const uint64_t* xp, uint64_t* dst,
                                            double* sm) {
  warp_lr_stream_body<NT2, LOGPDF>(tg, part, xp, dst, sm);
}
#endif

// does this machine stream target tg's design (warp_lr dispatch; codegen emits the same test)
__device__ __forceinline__ bool lr_streams(const DevTarget& tg, int sm_doubles) {
  return tg.n >= kLrStreamMinN && sm_doubles >= lr_stream_doubles(tg.dim);
}

// grad (want_logpdf = false) or fast logpdf of a logistic-regression target, DMMA path;
// sm_doubles: the warp's shared-memory scratch (tall designs stream through it)
__device__ inline void warp_lr(const DevTarget& tg, bool part, const uint64_t* xp, uint64_t* dst, double* Xs,
                               bool want_logpdf, int sm_doubles) {
  if (tg.n >= kLrStreamMinN && sm_doubles >= lr_stream_doubles(tg.dim)) {  // = lr_streams
    switch (tg.NT2) {
#define LSB_LRS_CASE(K)                                                        \
  case K:                                                                      \
    if (want_logpdf) warp_lr_stream<K, true>(tg, part, xp, dst, Xs);           \
    else warp_lr_stream<K, false>(tg, part, xp, dst, Xs);                      \
    return;
      LSB_LRS_CASE(1) LSB_LRS_CASE(2) LSB_LRS_CASE(3) LSB_LRS_CASE(4) LSB_LRS_CASE(5) LSB_LRS_CASE(6)
      LSB_LRS_CASE(7) LSB_LRS_CASE(8) LSB_LRS_CASE(9) LSB_LRS_CASE(10) LSB_LRS_CASE(11) LSB_LRS_CASE(12)
      LSB_LRS_CASE(13) LSB_LRS_CASE(14) LSB_LRS_CASE(15) LSB_LRS_CASE(16)
#undef LSB_LRS_CASE
      default: break;
    }
  }
  switch (tg.NT2) {
#define LSB_LR_CASE(K)                                                   \
  case K:                                                                \
    if (want_logpdf) warp_lr_nt<K, true>(tg, part, xp, dst, Xs);         \
    else warp_lr_nt<K, false>(tg, part, xp, dst, Xs);                    \
    return;
    LSB_LR_CASE(1) LSB_LR_CASE(2) LSB_LR_CASE(3) LSB_LR_CASE(4) LSB_LR_CASE(5) LSB_LR_CASE(6)
    LSB_LR_CASE(7) LSB_LR_CASE(8) LSB_LR_CASE(9) LSB_LR_CASE(10) LSB_LR_CASE(11) LSB_LR_CASE(12)
    LSB_LR_CASE(13) LSB_LR_CASE(14) LSB_LR_CASE(15) LSB_LR_CASE(16)
#undef LSB_LR_CASE
    default: break;
  }
}

__device__ inline void warp_lr_grad(const DevTarget& tg, bool part, const uint64_t* xp, uint64_t* dst,
                                    double* Xs) {
  warp_lr(tg, part, xp, dst, Xs, false, 0);
}

// LR gradients take the DMMA path when the warp's scratch holds an 8-chain tile of w
__device__ __forceinline__ bool lr_coop(const VMArgs& a, const DevTarget& tg) {
  return tg.kind == LS_TARGET_LOGREG && tg.NT2 <= 16 && 8 * lf_stride_q(tg.dim) <= a.lf_smem_per_warp;
}

__device__ __forceinline__ bool warp_coop(const VMArgs& a, const ROp& op) {
  if (op.opcode == LS_OP_GRAD)
    return a.targets[op.imm0].kind == LS_TARGET_GAUSSIAN || lr_coop(a, a.targets[op.imm0]);
  if (op.opcode == LS_OP_LOGPDF)
    return !a.exact_logpdf &&
           (a.targets[op.imm0].kind == LS_TARGET_GAUSSIAN || lr_coop(a, a.targets[op.imm0]));
  return false;
}

// Shared-memory row strides (doubles) of the superblock tiles: DMMA A-fragment
// loads (8 rows x 4 cols, 64-bit) and C-fragment epilogues (8 rows x 2 cols,
// 128-bit) are bank-conflict free.
__host__ __device__ __forceinline__ int lf_stride_p(int d) { int s = (d + 7) / 8 * 8; return s + ((8 - s % 16) + 16) % 16; }
// d <= 128 uses the register-momentum superblock (only q staged in shared memory): kLfRegMaxTiles
__host__ __device__ __forceinline__ int lf_smem_doubles(int d) {
  return (d + 7) / 8 <= kLfRegMaxTiles ? 8 * lf_stride_q(d) : 8 * (lf_stride_q(d) + lf_stride_p(d)) + 8;
}

// One accumulator pass (n-tiles C0 .. C0+7) of the register-momentum superblock:
// g = -(q P) for the tile's 8 chains, p += (e/2) g in the C-fragment layout.
// nkick = 2 applies the same gradient twice, as two separately rounded kicks: the last
// half-kick of leapfrog step i and the first of step i+1 contract the same q (the
// reference recomputes it, workloads.py:464-467), so a leaf costs L+1 contractions.
template <int NT, int C0, bool SB>
__device__ __forceinline__ void lf_kick(double (&p)[NT][2], const double* Qs, int SQ, const DevTarget& tg,
                                        const double* Bf, double half, bool last, uint64_t* gg, int d,
                                        bool want_lp, double& quad, int nkick) {
  // LSB_LF_KC n-tiles per pass: p (in registers) + acc + prefetched fragments fit
  constexpr int NTC = (NT - C0) < LSB_LF_KC ? (NT - C0) : LSB_LF_KC;
  const int lane = threadIdx.x & 31, g = lane >> 2;
  double acc[NTC][2];
  lsb::mtile_gemm_pf<NTC, SB>(acc, Bf, tg.KS1, tg.NT1, C0, [&](int k) -> double { return Qs[g * SQ + k]; });
#pragma unroll
  for (int j = 0; j < NTC; ++j) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double gv = -acc[j][e];
      p[C0 + j][e] = __dadd_rn(__dmul_rn(half, gv), p[C0 + j][e]);
      if (nkick == 2) p[C0 + j][e] = __dadd_rn(__dmul_rn(half, gv), p[C0 + j][e]);
      const int col = 8 * (C0 + j) + 2 * (lane & 3) + e;
      if (last && gg != nullptr && col < d) gg[(size_t)col * 32] = f64_bits(gv);
      // the last kick contracts at the final q: accumulate q.(P q) in warp_gauss's order
      if (last && want_lp && col < d) quad = fma(Qs[g * SQ + col], acc[j][e], quad);
    }
  }
}

// All passes of one kick: n-tiles C0, C0 + LSB_LF_KC, ... < NT.
template <int NT, int C0, bool SB>
__device__ __forceinline__ void lf_kicks(double (&p)[NT][2], const double* Qs, int SQ, const DevTarget& tg,
                                         const double* Bf, double half, bool last, uint64_t* gg, int d,
                                         bool want_lp, double& quad, int nkick) {
  lf_kick<NT, C0, SB>(p, Qs, SQ, tg, Bf, half, last, gg, d, want_lp, quad, nkick);
  if constexpr (C0 + LSB_LF_KC < NT)
    lf_kicks<NT, C0 + LSB_LF_KC, SB>(p, Qs, SQ, tg, Bf, half, last, gg, d, want_lp, quad, nkick);
}

// Dev-only phase clock of the superblock (-DLSB_SB_PROFILE=1; tools/sb_profile.py):
// [0] q staging, [1] p load, [2] kicks (DMMA), [3] drifts, [4] write-back, [5] calls
#if LSB_SB_PROFILE
__device__ unsigned long long lsb_sb_prof[8];
#define LSB_SB_T(v) const long long v = clock64()
#define LSB_SB_ADD(i, t0, t1) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&lsb_sb_prof[i], (unsigned long long)((t1) - (t0)))
#else
#define LSB_SB_T(v)
#define LSB_SB_ADD(i, t0, t1)
#endif

// Register-momentum variant of the fused leapfrog superblock (d <= 128): p lives in
// registers in the DMMA C-fragment layout, q in shared memory (A-fragment source).
// Half the shared-memory footprint of the tile version, which leaves room for the
// CTA-wide staged copy of the precision matrix's B fragments (Bf, SB = true).
// op.pad >= 0: also write the fast logpdf at the final q to that row (the
// caller's `logpdf(q1)`, lowering.fuse_leaf_logpdf), from the last kick's DMMAs.
template <int NT, bool SB>
__device__ void warp_leapfrog_rp(const VMArgs& a, const Lane& ln, const ROp& op, bool part, double* sm,
                                 long long chain, const double* Bf) {
  const int lane = threadIdx.x & 31, g = lane >> 2;
  const DevTarget& tg = a.targets[op.imm0];
  const int d = tg.dim, steps = op.imm1;
  const int SQ = lf_stride_q(d);
  double* Qs = sm;
  const int grow = (int)(op.bits & 0xffffffff), irow = (int)(op.bits >> 32);
  __syncwarp();
  const unsigned mask = __ballot_sync(kFull, part);
  const int n = __popc(mask);
  // q, p: the function's registers, or (forwarded) the caller's argument sources
  uint64_t* myq = part ? const_cast<uint64_t*>(ln.in(op, 0)) : nullptr;
  uint64_t* myp = part ? const_cast<uint64_t*>(ln.in(op, 1)) : nullptr;
  const bool wb = (op.kind & 1) != 0;  // q, p read after the return: write them back
  const bool want_lp = op.pad >= 0;
  uint64_t* my_lp = (part && want_lp) ? ln.row(op.pad) : nullptr;
  const double mye = part ? as_f64(ln.in(op, 2)[0]) : 0.0;
  uint64_t* my_g = (part && grow >= 0) ? ln.row(grow) : nullptr;
  uint64_t* my_ret = part ? ln.row(op.out_row) : nullptr;
  if (part && irow >= 0) ln.row(irow)[0] = (uint64_t)(int64_t)steps;
  if (part && a.lane_trace != nullptr) {
    const int head = op.imm2;
    lane_trace_put(a, chain, head);
    for (int i = 0; i < steps; ++i) {
      lane_trace_put(a, chain, head + 1);
      lane_trace_put(a, chain, head);
    }
    lane_trace_put(a, chain, head + 2);
  }
  for (int mt = 0; mt * 8 < n; ++mt) {
    LSB_SB_T(t_a);
    stage_mtile<(8 * NT + 16 + 3) / 4>(Qs, SQ, myq, mask, n, mt, d);  // q of the m-tile's 8 chains, one round trip
    LSB_SB_T(t_b);
    LSB_SB_ADD(0, t_a, t_b);
    const int src = mtile_lane(mask, n, mt, g);
    const int sl = src < 0 ? 0 : src;
    const uint64_t* pg = (const uint64_t*)__shfl_sync(kFull, (unsigned long long)myp, sl);
    const double eg = __shfl_sync(kFull, mye, sl);
    uint64_t* gg = (uint64_t*)__shfl_sync(kFull, (unsigned long long)my_g, sl);
    if (src < 0) gg = nullptr;
    const double half = __ddiv_rn(eg, 2.0);
    double quad = 0.0;
    double p[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 8 * nt + 2 * (lane & 3) + e;
        p[nt][e] = (src >= 0 && col < d) ? as_f64(pg[(size_t)col * 32]) : 0.0;
      }
    __syncwarp();
#if LSB_SB_PROFILE
    if (p[0][0] == 123.456) p[0][1] = 0.0;  // force the p loads to complete here
#endif
    LSB_SB_T(t_c);
    LSB_SB_ADD(1, t_b, t_c);
    // L+1 contractions: g(q0) then, per step, drift and g(q_{i+1}), whose kick serves
    // the end of step i and the start of step i+1 (two separately rounded kicks)
    if (steps > 0) {
      LSB_SB_T(t_k0);
      lf_kicks<NT, 0, SB>(p, Qs, SQ, tg, Bf, half, false, gg, d, want_lp, quad, 1);
      __syncwarp();
      LSB_SB_T(t_k1);
      LSB_SB_ADD(2, t_k0, t_k1);
    }
    for (int it = 0; it < steps; ++it) {
      LSB_SB_T(t_d0);
      // drift: q = e p + q on this thread's (row, columns)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * nt + 2 * (lane & 3) + e;
          if (col < d) Qs[g * SQ + col] = __dadd_rn(__dmul_rn(eg, p[nt][e]), Qs[g * SQ + col]);
        }
      __syncwarp();
      LSB_SB_T(t_d1);
      LSB_SB_ADD(3, t_d0, t_d1);
      const bool last = it == steps - 1;
      lf_kicks<NT, 0, SB>(p, Qs, SQ, tg, Bf, half, last, gg, d, want_lp, quad, last ? 1 : 2);
      __syncwarp();
      LSB_SB_T(t_k2);
      LSB_SB_ADD(2, t_d1, t_k2);
    }
    if (want_lp) {  // warp_gauss's reduction over the row's 4 threads
      quad += __shfl_xor_sync(kFull, quad, 1);
      quad += __shfl_xor_sync(kFull, quad, 2);
      uint64_t* lo = (uint64_t*)__shfl_sync(kFull, (unsigned long long)my_lp, sl);
      if (src >= 0 && (lane & 3) == 0) lo[0] = f64_bits(gauss_lp_from_quad(tg.norm, quad));
    }
    LSB_SB_T(t_w0);
    // write back q, p and _ret = vcat(q, p): each thread its (row, columns)
    uint64_t* qo = (uint64_t*)__shfl_sync(kFull, (unsigned long long)myq, sl);
    uint64_t* po = (uint64_t*)__shfl_sync(kFull, (unsigned long long)myp, sl);
    uint64_t* ro = (uint64_t*)__shfl_sync(kFull, (unsigned long long)my_ret, sl);
    if (src >= 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * nt + 2 * (lane & 3) + e;
          if (col < d) {
            const uint64_t qv = f64_bits(Qs[g * SQ + col]), pv = f64_bits(p[nt][e]);
            if (wb) {
              qo[(size_t)col * 32] = qv;
              po[(size_t)col * 32] = pv;
            }
            ro[(size_t)col * 32] = qv;
            ro[(size_t)(d + col) * 32] = pv;
          }
        }
    }
    __syncwarp();
    LSB_SB_T(t_w1);
    LSB_SB_ADD(4, t_w0, t_w1);
  }
#if LSB_SB_PROFILE
  if (lane == 0) atomicAdd(&lsb_sb_prof[5], 1ull);
#endif
}

// Fused leapfrog superblock: the whole `leapfrog(q, p, e)` function of the
// NUTS-lite program (reference workloads.py:461-472; flat blocks
// leapfrog.b0..b3) for every participating lane, run to return, with q and p
// resident in shared memory across all 2L gradient contractions:
//   repeat L: g = -(q P); p = (e/2) g + p; q = e p + q; g = -(q P); p = (e/2) g + p
// Every update is the reference's separate IEEE multiply then add (axpy,
// runtime.py:253-255); e/2 is the reference's `div e 2.0`. Writes back
// leapfrog.{q, p, g, i, _ret}; the block's terminator pops the pc (return).
// op: in = {q, p, e}, out row = _ret, imm0 = target slot, imm1 = L,
//     imm2 = loop-head block, bits = g_row | i_row << 32.
template <bool SB>
__device__ void warp_leapfrog_tile(const VMArgs& a, const Lane& ln, const ROp& op, bool part, double* sm,
                                   long long chain, const double* Bf);

// One out-of-line register-momentum superblock for a target with NT n-tiles
// (program-specialised builds call this directly: one compact body in the i-cache).
#ifndef LSB_SB_INLINE
#define LSB_SB_INLINE 0
#endif
#if LSB_SB_INLINE
#define LSB_SB_QUAL __forceinline__
#else
#define LSB_SB_QUAL __noinline__
#endif
#include "lsb_tc_leapfrog.cuh"

template <int NT>
__device__ LSB_SB_QUAL void warp_leapfrog_nt(const VMArgs& a, const Lane ln, const ROp op, bool part,
                                              double* sm, long long chain) {
  if (a.tc_img != nullptr) {  // fp32 arm: the warpgroup's 128 chains on tcgen05
    if constexpr (NT <= 16) wg_leapfrog_tf32<NT>(a, ln, op, part, chain);
    return;
  }
  const double* Bs = staged_B(a, op.imm0);
  if (Bs) warp_leapfrog_rp<NT, true>(a, ln, op, part, sm, chain, Bs);
  else warp_leapfrog_rp<NT, false>(a, ln, op, part, sm, chain, a.targets[op.imm0].B1);
}

__device__ inline void warp_leapfrog(const VMArgs& a, const Lane& ln, const ROp& op, bool part, double* sm,
                                     long long chain) {
  if (a.tc_img != nullptr) {
    wg_leapfrog_tf32_any(a, ln, op, part, chain);
    return;
  }
  const DevTarget& tg = a.targets[op.imm0];
  const double* Bs = staged_B(a, op.imm0);
  switch (tg.NT1) {  // d <= 128: register-momentum variant
#define LSB_LF_CASE(K)                                                         \
  case K:                                                                      \
    if (Bs) warp_leapfrog_rp<K, true>(a, ln, op, part, sm, chain, Bs);         \
    else warp_leapfrog_rp<K, false>(a, ln, op, part, sm, chain, tg.B1);        \
    return;
    LSB_LF_CASE(1) LSB_LF_CASE(2) LSB_LF_CASE(3) LSB_LF_CASE(4) LSB_LF_CASE(5) LSB_LF_CASE(6)
    LSB_LF_CASE(7) LSB_LF_CASE(8) LSB_LF_CASE(9) LSB_LF_CASE(10) LSB_LF_CASE(11) LSB_LF_CASE(12)
    LSB_LF_CASE(13) LSB_LF_CASE(14) LSB_LF_CASE(15) LSB_LF_CASE(16)
#undef LSB_LF_CASE
    default: break;
  }
  if (Bs) warp_leapfrog_tile<true>(a, ln, op, part, sm, chain, Bs);
  else warp_leapfrog_tile<false>(a, ln, op, part, sm, chain, tg.B1);
}

template <bool SB>
__device__ void warp_leapfrog_tile(const VMArgs& a, const Lane& ln, const ROp& op, bool part, double* sm,
                                   long long chain, const double* Bf) {
  const int lane = threadIdx.x & 31;
  const DevTarget& tg = a.targets[op.imm0];
  const int d = tg.dim, steps = op.imm1;
  const int SQ = lf_stride_q(d), SP = lf_stride_p(d);
  double* Qs = sm;
  double* Ps = sm + 8 * SQ;
  double* Es = Ps + 8 * SP;
  const int grow = (int)(op.bits & 0xffffffff), irow = (int)(op.bits >> 32);
  __syncwarp();
  const unsigned mask = __ballot_sync(kFull, part);
  const int n = __popc(mask);
  uint64_t* myq = part ? const_cast<uint64_t*>(ln.in(op, 0)) : nullptr;
  uint64_t* myp = part ? const_cast<uint64_t*>(ln.in(op, 1)) : nullptr;
  const bool wb = (op.kind & 1) != 0;
  const double mye = part ? as_f64(ln.in(op, 2)[0]) : 0.0;
  uint64_t* my_g = (part && grow >= 0) ? ln.row(grow) : nullptr;
  uint64_t* my_ret = part ? ln.row(op.out_row) : nullptr;
  if (part && irow >= 0) ln.row(irow)[0] = (uint64_t)(int64_t)steps;
  if (part && a.lane_trace != nullptr) {  // the blocks a lane walks inside the function
    const int head = op.imm2;
    lane_trace_put(a, chain, head);
    for (int i = 0; i < steps; ++i) {
      lane_trace_put(a, chain, head + 1);
      lane_trace_put(a, chain, head);
    }
    lane_trace_put(a, chain, head + 2);
  }
  for (int mt = 0; mt * 8 < n; ++mt) {
    for (int r = 0; r < 8; ++r) {  // stage the m-tile's 8 chains (zero rows pad)
      const int lr = mtile_lane(mask, n, mt, r);
      const uint64_t* qg = (const uint64_t*)__shfl_sync(kFull, (unsigned long long)myq, lr < 0 ? 0 : lr);
      const uint64_t* pg = (const uint64_t*)__shfl_sync(kFull, (unsigned long long)myp, lr < 0 ? 0 : lr);
      const double er = __shfl_sync(kFull, mye, lr < 0 ? 0 : lr);
      for (int k = lane; k < SQ; k += 32) Qs[r * SQ + k] = (lr >= 0 && k < d) ? as_f64(qg[(size_t)k * 32]) : 0.0;
      for (int k = lane; k < SP; k += 32) Ps[r * SP + k] = (lr >= 0 && k < d) ? as_f64(pg[(size_t)k * 32]) : 0.0;
      if (lane == 0) Es[r] = lr >= 0 ? er : 0.0;
    }
    __syncwarp();
    const int g = lane >> 2;
    const int src = mtile_lane(mask, n, mt, g);
    const double half = __ddiv_rn(Es[g], 2.0);
    uint64_t* gg = (uint64_t*)__shfl_sync(kFull, (unsigned long long)my_g, src < 0 ? 0 : src);
    auto a_at = [&](int k) -> double { return Qs[g * SQ + k]; };
    // L+1 contractions (see lf_kick): pass 0 kicks with g(q0); pass i >= 1 drifts, then
    // kicks twice with g(q_i) (end of step i-1, start of step i), once on the last pass
    for (int pass = 0; steps > 0 && pass <= steps; ++pass) {
      if (pass > 0) {  // q = e p + q over the tile
        for (int idx = lane; idx < 8 * d; idx += 32) {
          const int r = idx / d, k = idx - r * d;
          Qs[r * SQ + k] = __dadd_rn(__dmul_rn(Es[r], Ps[r * SP + k]), Qs[r * SQ + k]);
        }
        __syncwarp();
      }
      const bool last = pass == steps;
      const int nkick = (pass == 0 || last) ? 1 : 2;
      for (int nt0 = 0; nt0 < tg.NT1; nt0 += LSB_NT_CHUNK) {
        const int ntc = min(LSB_NT_CHUNK, tg.NT1 - nt0);
        LSB_NT_DISPATCH(ntc, {
          double acc[NTC][2];
          lsb::mtile_gemm<NTC, SB>(acc, Bf, tg.KS1, tg.NT1, nt0, a_at);
          _Pragma("unroll")
          for (int j = 0; j < NTC; ++j) {
            const int col = 8 * (nt0 + j) + 2 * (lane & 3);
            double2* pp = reinterpret_cast<double2*>(Ps + g * SP + col);
            double2 pv = *pp;
            const double g0 = -acc[j][0], g1 = -acc[j][1];
            pv.x = __dadd_rn(__dmul_rn(half, g0), pv.x);
            pv.y = __dadd_rn(__dmul_rn(half, g1), pv.y);
            if (nkick == 2) {
              pv.x = __dadd_rn(__dmul_rn(half, g0), pv.x);
              pv.y = __dadd_rn(__dmul_rn(half, g1), pv.y);
            }
            if (col + 1 < d) *pp = pv;
            else if (col < d) Ps[g * SP + col] = pv.x;  // odd d: the pad column stays zero
            if (last && src >= 0 && gg != nullptr) {
              if (col < d) gg[(size_t)col * 32] = f64_bits(g0);
              if (col + 1 < d) gg[(size_t)(col + 1) * 32] = f64_bits(g1);
            }
          }
        });
      }
      __syncwarp();
    }
    for (int r = 0; r < 8; ++r) {  // write back q, p and _ret = vcat(q, p)
      const int lr = mtile_lane(mask, n, mt, r);
      if (lr < 0) break;
      uint64_t* qo = (uint64_t*)__shfl_sync(kFull, (unsigned long long)myq, lr);
      uint64_t* po = (uint64_t*)__shfl_sync(kFull, (unsigned long long)myp, lr);
      uint64_t* ro = (uint64_t*)__shfl_sync(kFull, (unsigned long long)my_ret, lr);
      for (int k = lane; k < d; k += 32) {
        const uint64_t qv = f64_bits(Qs[r * SQ + k]), pv = f64_bits(Ps[r * SP + k]);
        if (wb) {
          qo[(size_t)k * 32] = qv;
          po[(size_t)k * 32] = pv;
        }
        ro[(size_t)k * 32] = qv;
        ro[(size_t)(d + k) * 32] = pv;
      }
    }
    __syncwarp();
  }
}

// ---- one block step for one lane (both engines) ---------------------------------------------

struct StepFault {
  int pos = 0;  // op position + 1 (0 = none)
  int kind = 0, var = 0, detail = 0;
};

// Execute block `b` for this lane (if active). WARP selects the warp-group
// engine (cooperative DMMA ops and superblocks; every thread of the warp must
// call). Returns true when the lane's pc reached the halt block.
template <bool WARP>
__device__ __forceinline__ bool exec_block(const VMArgs& a, const Lane& ln, int b, bool active,
                                           long long chain, StepFault& f, double* lf_smem) {
  const RBlock blk = a.blocks[b];
  const ROp* ops = a.ops + blk.op_begin;
  for (int k = 0; k < blk.op_count; ++k) {
    const ROp& op = ops[k];
    if (op.opcode == LS_OP_LEAPFROG) {
      if constexpr (WARP) warp_leapfrog(a, ln, op, active && !f.pos, lf_smem, chain);
      continue;
    }
    const bool coop = WARP && warp_coop(a, op);
    if (!coop && (!active || f.pos)) continue;
    bool part = active && !f.pos;
    uint64_t* dst = nullptr;
    bool push = false;
    if (part) {
      if (op.action == LS_POP) {
        int& s = ln.sp_row(op.out_sp);
        if (s < 1) f = StepFault{k + 1, LS_RUN_UNDERFLOW, op.out, 0};
        else --s;
        part = false;
      } else if (op.out_sp >= 0) {
        const int s = ln.sp_row(op.out_sp);
        if (op.action == LS_PUSH) {
          if (s >= a.depth) { f = StepFault{k + 1, LS_RUN_OVERFLOW, op.out, 0}; part = false; }
          else { dst = ln.row(op.out_row + s * op.width); push = true; }
        } else if (s < 1) {
          f = StepFault{k + 1, LS_RUN_UNDERFLOW, op.out, 1};
          part = false;
        } else {
          dst = ln.row(op.out_row + (s - 1) * op.width);
        }
      } else {
        dst = ln.row(op.out_row);
      }
    }
    if (coop) {
      if constexpr (WARP) {
        __syncwarp();
        if (a.targets[op.imm0].kind == LS_TARGET_LOGREG)
          warp_lr(a.targets[op.imm0], part, part ? ln.in(op, 0) : nullptr, dst, lf_smem,
                  op.opcode == LS_OP_LOGPDF, a.lf_smem_per_warp);
        else
          warp_gauss(a.targets[op.imm0], staged_B(a, op.imm0), part, part ? ln.in(op, 0) : nullptr, dst,
                     op.opcode == LS_OP_LOGPDF, lf_smem, a.lf_smem_per_warp);
        __syncwarp();
      }
    } else if (part && op.opcode != LS_OP_ALLOC) {  // alloc: the slot is reserved, not written
      compute_op(a, op, op.nin > 0 ? ln.in(op, 0) : nullptr, op.nin > 1 ? ln.in(op, 1) : nullptr,
                 op.nin > 2 ? ln.in(op, 2) : nullptr, dst, ln.L);
    }
    if (part && push) ++ln.sp_row(op.out_sp);
  }
  if (!active || f.pos) return false;
  int& psp = ln.sp_row(a.n_sp_rows - 1);
  int* top = &ln.pcs[(psp - 1) * ln.L + ln.t];
  switch (blk.term) {
    case LS_JUMP: *top = blk.a; break;
    case LS_BRANCH: *top = (ln.top(blk.cond_row, blk.cond_sp, blk.cond_w)[0] != 0) ? blk.a : blk.b; break;
    case LS_PUSHJUMP:
      *top = blk.b;
      if (psp >= a.depth + 1) {
        f = StepFault{blk.op_count + 1, LS_RUN_OVERFLOW, -1, 0};
      } else {
        ln.pcs[psp * ln.L + ln.t] = blk.a;
        ++psp;
      }
      break;
    default:
      if (psp < 1) {
        f = StepFault{blk.op_count + 1, LS_RUN_UNDERFLOW, -1, 0};
      } else {
        --psp;
        if (psp >= 1 && ln.pcs[(psp - 1) * ln.L + ln.t] == a.halt) return true;
      }
      break;
  }
  return false;
}

}  // namespace lsbvm
