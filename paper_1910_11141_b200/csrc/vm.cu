// vm.cu — the B200 program-counter VM (paper Alg. 2 / reference pc_vm.py).
//
// Execution model
//   * One CTA is one autobatching group: blockDim.x lanes, one thread per
//     lane. Every step the CTA builds the program-counter histogram of its
//     live lanes (warp __match_any_sync + popc into shared counters, or a
//     warp min-reduction for the reference's min-pc rule), selects one block,
//     and the threads whose pc sits at that block execute it. Lanes are
//     independent (reference runtime.py:96-104), so groups need no grid-wide
//     synchronisation and per-lane results do not depend on the schedule.
//   * The kernel is persistent and resumable: all machine state (data
//     stacks, stack pointers, pc stacks, registers, scratch) lives in a
//     per-group HBM workspace in lane-minor layout, so a launch can stop
//     after any step and the next launch continues.
//   * When Z exceeds one group, groups pull chains from a global counter and
//     refill a lane slot as soon as its chain halts (continuous batching).
//   * Faults (stack overflow/underflow) are reported as the lowest
//     (op position, lane) of the faulting step, like reference
//     runtime.py:462-507; the whole machine stops (no rollback).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lockstep_b200.h"
#include "lsb_ops.cuh"
#include "lsb_leapfrog.cuh"

using lsb::as_f64;
using lsb::f64_bits;

namespace {

constexpr int kMaxTargets = 8;
constexpr int kMaxLanes = 1024;

struct DevTarget {
  int kind = 0, dim = 0, n = 0;
  const double* P = nullptr;   // gaussian: precision (d x d, row-major); logreg: sx (n x d)
  const double* PT = nullptr;  // transpose of the above
  double norm = 0.0;
};

struct FaultRec {
  unsigned long long key;  // (op position << 32) | lane-in-group, min wins
  int kind;                // LS_RUN_OVERFLOW / LS_RUN_UNDERFLOW
  int var;                 // -1 = pc stack
  int block;
  int detail;              // 1 = underflow of an update (write_top)
  long long chain;
};

struct VMArgs {
  // program
  const ls_block* blocks;
  const ls_op* ops;
  const ls_var* vars;
  const int* var_row;       // first workspace row of each var
  const int* var_depth;     // slots of each var (depth for stacked, else 1)
  int n_blocks, halt, entry;
  int n_inputs;
  const int* input_vars;
  int output_var;
  int n_sp_rows;            // stacked vars + 1 (pc)
  DevTarget targets[kMaxTargets];
  // machine
  long long z;
  int depth;
  int lanes;                // == blockDim.x
  int group_rows;           // workspace rows per group
  uint64_t* ws;
  int* sp;                  // [groups][n_sp_rows][lanes]
  int* pcs;                 // [groups][depth+1][lanes]
  long long* chain_of;      // [groups][lanes]  (-1 free, -2 exhausted)
  const uint64_t* const* inputs;  // device arrays [z][width]
  const int* input_width;
  uint64_t* output;         // [z][out_width]
  int out_width;
  unsigned long long* next_chain;
  int refill;
  int sched;
  int exact_logpdf;
  long long max_steps;      // <0 unbounded (StepLimitExceeded bound, per group)
  long long* group_steps;   // [groups]
  int* group_done;          // [groups]
  // observability
  int* trace_block;         // single-group trace
  int* trace_active;
  long long trace_cap;
  long long* trace_n;
  long long* blk_steps;     // [groups][n_blocks]
  long long* blk_active;    // [groups][n_blocks]
  unsigned long long* useful;
  unsigned long long* launched;
  int* lane_trace;          // [z][lane_trace_cap] per-chain block sequence (debug/parity)
  int* lane_trace_len;      // [z]
  int lane_trace_cap;
  FaultRec* fault;
  int* abort_flag;
  int* paused;
};

struct Lane {
  const VMArgs* a;
  uint64_t* ws;   // group workspace
  int* sp;        // group stack pointers
  int* pcs;       // group pc stack
  int t, L;

  __device__ __forceinline__ uint64_t* row(int r) const { return ws + (size_t)r * L + t; }
  __device__ __forceinline__ int& sp_of(int v) const { return sp[a->vars[v].sp * L + t]; }
  // base pointer of the var's current top slot (junk slot 0 for empty stacks)
  __device__ __forceinline__ uint64_t* top(int v) const {
    const ls_var& vd = a->vars[v];
    int slot = 0;
    if (vd.cls == LS_STACKED) {
      slot = sp_of(v) - 1;
      if (slot < 0) slot = 0;
    }
    return row(a->var_row[v] + slot * vd.width);
  }
  __device__ __forceinline__ uint64_t* slot_ptr(int v, int slot) const {
    return row(a->var_row[v] + slot * a->vars[v].width);
  }
};

__device__ __forceinline__ int64_t as_i64_any(uint64_t w, int kind) {
  return kind == LS_F64 ? lsb::f64_to_i64(as_f64(w)) : (int64_t)w;
}

// ---- target densities ---------------------------------------------------------------

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

__device__ double target_logpdf(const DevTarget& tg, const uint64_t* x, int stride, int exact) {
  if (tg.kind == LS_TARGET_GAUSSIAN) {
    if (exact) return lsb::gauss_logpdf_exact(x, stride, tg.dim, tg.P, tg.norm);
    // fused form: norm - 0.5 * sum_j x_j (P x)_j
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

__device__ void target_grad(const DevTarget& tg, const uint64_t* x, int stride, uint64_t* out) {
  const int d = tg.dim;
  if (tg.kind == LS_TARGET_GAUSSIAN) {
    // g_j = -(sum_i x_i P_ij): P^T rows are contiguous
    for (int j = 0; j < d; ++j) {
      const double* col = tg.PT + (size_t)j * d;
      double acc = 0.0;
      for (int i = 0; i < d; ++i) acc = fma(as_f64(x[(size_t)i * stride]), __ldg(col + i), acc);
      out[(size_t)j * stride] = f64_bits(-acc);
    }
    return;
  }
  // logistic: g = sig(m) @ sx - w, m = w @ sx^T
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

// ---- one primitive for one lane ----------------------------------------------------------

// Computes op into dst (width op.width words, lane stride L). Inputs are read
// through Lane::top, i.e. the current top slot of each input variable.
__device__ void compute_op(const Lane& ln, const ls_op& op, uint64_t* dst) {
  const VMArgs& a = *ln.a;
  const int L = ln.L;
  const int w = op.width;
  const uint64_t* x = op.nin > 0 ? ln.top(op.in[0]) : nullptr;
  const uint64_t* y = op.nin > 1 ? ln.top(op.in[1]) : nullptr;
  const uint64_t* u = op.nin > 2 ? ln.top(op.in[2]) : nullptr;
  const bool f = op.kind == LS_F64;
#define EACH for (int i = 0; i < w; ++i)
#define X(i) x[(size_t)(i) * L]
#define Y(i) y[(size_t)(i) * L]
#define D(i) dst[(size_t)(i) * L]
  switch (op.opcode) {
    case LS_OP_CONST: D(0) = (uint64_t)op.bits; break;
    case LS_OP_ID: EACH D(i) = X(i); break;
    case LS_OP_ADD:
      EACH D(i) = f ? f64_bits(__dadd_rn(as_f64(X(i)), as_f64(Y(i)))) : X(i) + Y(i);
      break;
    case LS_OP_SUB:
      EACH D(i) = f ? f64_bits(__dsub_rn(as_f64(X(i)), as_f64(Y(i)))) : X(i) - Y(i);
      break;
    case LS_OP_MUL:
      EACH D(i) = f ? f64_bits(__dmul_rn(as_f64(X(i)), as_f64(Y(i))))
                    : (uint64_t)((unsigned long long)X(i) * (unsigned long long)Y(i));
      break;
    case LS_OP_DIV:
      EACH {
        if (f) {
          D(i) = f64_bits(__ddiv_rn(as_f64(X(i)), as_f64(Y(i))));
        } else {  // numpy floor_divide on int64; division by zero yields 0
          const int64_t p = (int64_t)X(i), q = (int64_t)Y(i);
          int64_t r;
          if (q == 0) r = 0;
          else if (q == -1) r = (int64_t)(0ull - (uint64_t)p);
          else {
            r = p / q;
            if ((p % q != 0) && ((p < 0) != (q < 0))) r -= 1;
          }
          D(i) = (uint64_t)r;
        }
      }
      break;
    case LS_OP_MIN:
    case LS_OP_MAX: {
      const bool mn = op.opcode == LS_OP_MIN;
      EACH {
        if (f) {
          const double p = as_f64(X(i)), q = as_f64(Y(i));
          double r;
          if (p != p) r = p;
          else if (q != q) r = q;
          else r = mn ? (p <= q ? p : q) : (p >= q ? p : q);
          D(i) = f64_bits(r);
        } else {
          const int64_t p = (int64_t)X(i), q = (int64_t)Y(i);
          D(i) = (uint64_t)(mn ? (p < q ? p : q) : (p > q ? p : q));
        }
      }
      break;
    }
    case LS_OP_LE:
      D(0) = f ? (as_f64(X(0)) <= as_f64(Y(0))) : ((int64_t)X(0) <= (int64_t)Y(0));
      break;
    case LS_OP_LT:
      D(0) = f ? (as_f64(X(0)) < as_f64(Y(0))) : ((int64_t)X(0) < (int64_t)Y(0));
      break;
    case LS_OP_EQ:
      D(0) = f ? (as_f64(X(0)) == as_f64(Y(0))) : (X(0) == Y(0));
      break;
    case LS_OP_AND: D(0) = (X(0) != 0) && (Y(0) != 0); break;
    case LS_OP_OR: D(0) = (X(0) != 0) || (Y(0) != 0); break;
    case LS_OP_NOT: D(0) = X(0) == 0; break;
    case LS_OP_NEG:
      EACH D(i) = f ? f64_bits(-as_f64(X(i))) : (uint64_t)(0ull - X(i));
      break;
    case LS_OP_ABS:
      EACH {
        if (f) D(i) = f64_bits(fabs(as_f64(X(i))));
        else { const int64_t p = (int64_t)X(i); D(i) = p < 0 ? (uint64_t)(0ull - (uint64_t)p) : (uint64_t)p; }
      }
      break;
    case LS_OP_SQRT: EACH D(i) = f64_bits(__dsqrt_rn(as_f64(X(i)))); break;
    case LS_OP_EXP: EACH D(i) = f64_bits(exp(as_f64(X(i)))); break;
    case LS_OP_LOG: EACH D(i) = f64_bits(log(as_f64(X(i)))); break;
    case LS_OP_SIN: EACH D(i) = f64_bits(sin(as_f64(X(i)))); break;
    case LS_OP_COS: EACH D(i) = f64_bits(cos(as_f64(X(i)))); break;
    case LS_OP_FLOOR: EACH D(i) = f64_bits(floor(as_f64(X(i)))); break;
    case LS_OP_SELECT: {
      const bool c = X(0) != 0;
      const uint64_t* src = c ? y : u;
      EACH D(i) = src[(size_t)i * L];
      break;
    }
    case LS_OP_DOT: D(0) = f64_bits(lsb::dot_lane(x, y, a.vars[op.in[0]].width, L)); break;
    case LS_OP_AXPY: {
      const double s = as_f64(X(0));
      EACH D(i) = f64_bits(__dadd_rn(__dmul_rn(s, as_f64(Y(i))), as_f64(u[(size_t)i * L])));
      break;
    }
    case LS_OP_VGET: {
      const int vw = a.vars[op.in[0]].width;
      int64_t k = as_i64_any(Y(0), a.vars[op.in[1]].kind);
      k = k < 0 ? 0 : (k > vw - 1 ? vw - 1 : k);
      D(0) = X(k);
      break;
    }
    case LS_OP_VSTORE: {
      int64_t k = as_i64_any(Y(0), a.vars[op.in[1]].kind);
      k = k < 0 ? 0 : (k > w - 1 ? w - 1 : k);
      const uint64_t val = u[0];
      if (dst != x) EACH D(i) = X(i);
      D(k) = val;
      break;
    }
    case LS_OP_VCAT: {
      const int wa = a.vars[op.in[0]].width;
      if (dst != x) for (int i = 0; i < wa; ++i) D(i) = X(i);
      for (int i = wa; i < w; ++i) D(i) = Y(i - wa);
      break;
    }
    case LS_OP_VFILL: EACH D(i) = X(0); break;
    case LS_OP_VSLICE: EACH D(i) = X(op.imm0 + i); break;
    case LS_OP_RNG: {
      const int64_t k = as_i64_any(X(0), a.vars[op.in[0]].kind);
      const int64_t c = as_i64_any(Y(0), a.vars[op.in[1]].kind);
      D(0) = f64_bits(lsb::rng_uniform(k, c));
      break;
    }
    case LS_OP_LOGPDF:
      D(0) = f64_bits(target_logpdf(a.targets[op.imm0], x, L, a.exact_logpdf));
      break;
    case LS_OP_GRAD: target_grad(a.targets[op.imm0], x, L, dst); break;
    default: break;
  }
#undef EACH
#undef X
#undef Y
#undef D
}

__device__ __forceinline__ void record_fault(const VMArgs& a, unsigned long long* s_key, int pos, int t) {
  atomicMin(s_key, ((unsigned long long)pos << 32) | (unsigned)t);
}

// Copy the lane's output (top slot of the output var) into output[chain].
__device__ void write_output(const VMArgs& a, const Lane& ln, long long chain) {
  const uint64_t* src = ln.top(a.output_var);
  uint64_t* dst = a.output + (size_t)chain * a.out_width;
  for (int i = 0; i < a.out_width; ++i) dst[i] = src[(size_t)i * ln.L];
}

__device__ void init_lane(const VMArgs& a, const Lane& ln, long long chain) {
  // data stacks hold one live slot from the start (pc_vm.py:180-181)
  for (int r = 0; r + 1 < a.n_sp_rows; ++r) ln.sp[r * ln.L + ln.t] = 1;
  for (int k = 0; k < a.n_inputs; ++k) {
    const int v = a.input_vars[k];
    const int w = a.input_width[k];
    const uint64_t* src = a.inputs[k] + (size_t)chain * w;
    uint64_t* dst = ln.slot_ptr(v, 0);
    for (int i = 0; i < w; ++i) dst[(size_t)i * ln.L] = src[i];
  }
  // pc stack seeded [halt, entry], pointer 2 (pc_vm.py:199-203)
  ln.pcs[0 * ln.L + ln.t] = a.halt;
  ln.pcs[1 * ln.L + ln.t] = a.entry;
  ln.sp[(a.n_sp_rows - 1) * ln.L + ln.t] = 2;
}

struct SchedShared {
  int pick;
  int count;
  unsigned long long fault_key;
  int any_live;
  int warp_val[kMaxLanes / 32];
  int warp_cnt[kMaxLanes / 32];
};

__global__ void __launch_bounds__(kMaxLanes) vm_kernel(const __grid_constant__ VMArgs a) {
  extern __shared__ int s_hist[];  // [n_blocks + 1]
  __shared__ SchedShared sh;
  __shared__ LeapfrogShared lf_shared;

  const int g = blockIdx.x;
  const int t = threadIdx.x;
  const int L = a.lanes;
  const int lane_id = t & 31, warp = t >> 5, nwarps = (L + 31) >> 5;
  Lane ln{&a, a.ws + (size_t)g * a.group_rows * L, a.sp + (size_t)g * a.n_sp_rows * L,
          a.pcs + (size_t)g * (a.depth + 1) * L, t, L};
  int* pc_sp = ln.sp + (a.n_sp_rows - 1) * L + t;
  long long* my_chain = a.chain_of + (size_t)g * L + t;
  long long steps = a.group_steps[g];
  long long* bsteps = a.blk_steps + (size_t)g * a.n_blocks;
  long long* bactive = a.blk_active + (size_t)g * a.n_blocks;
  unsigned long long useful = 0, launched = 0;

  if (a.group_done[g]) return;

  for (;;) {
    // ---- refill free lane slots from the global chain queue
    if (a.refill && *my_chain == -1) {
      const unsigned long long c = atomicAdd(a.next_chain, 1ull);
      if ((long long)c < a.z) {
        *my_chain = (long long)c;
        init_lane(a, ln, (long long)c);
      } else {
        *my_chain = -2;
      }
    }
    const bool has = *my_chain >= 0;
    const int pc = has ? ln.pcs[(*pc_sp - 1) * L + t] : a.halt;

    // ---- select the block (pc histogram / min reduction)
    if (t == 0) { sh.fault_key = ~0ull; }
    if (a.sched == LS_SCHED_MOST_POPULATED) {
      for (int b = t; b <= a.n_blocks; b += L) s_hist[b] = 0;
      __syncthreads();
      const unsigned peers = __match_any_sync(0xffffffffu, pc);
      if (pc != a.halt && lane_id == __ffs(peers) - 1) atomicAdd(&s_hist[pc], __popc(peers));
      __syncthreads();
      // argmax over blocks, ties to the lowest index
      int best = -1, best_b = a.halt;
      for (int b = t; b < a.n_blocks; b += L) {
        const int c = s_hist[b];
        if (c > best) { best = c; best_b = b; }
      }
      unsigned long long key = best > 0 ? (((unsigned long long)(unsigned)best) << 32) |
                                              (unsigned)(0x7fffffff - best_b) : 0ull;
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other > key ? other : key;
      }
      if (lane_id == 0) {
        sh.warp_val[warp] = (int)(key >> 32);
        sh.warp_cnt[warp] = (int)(0x7fffffff - (int)(key & 0xffffffffu));
      }
      __syncthreads();
      if (t == 0) {
        int bc = 0, bb = a.halt;
        for (int w2 = 0; w2 < nwarps; ++w2) {
          const int c = sh.warp_val[w2], b = sh.warp_cnt[w2];
          if (c > bc || (c == bc && c > 0 && b < bb)) { bc = c; bb = b; }
        }
        sh.pick = bc > 0 ? bb : a.halt;
        sh.count = bc;
      }
      __syncthreads();
    } else {
      const int m = __reduce_min_sync(0xffffffffu, (unsigned)pc);
      if (lane_id == 0) sh.warp_val[warp] = m;
      __syncthreads();
      if (t == 0) {
        int mm = a.halt;
        for (int w2 = 0; w2 < nwarps; ++w2) mm = min(mm, sh.warp_val[w2]);
        sh.pick = mm;
      }
      __syncthreads();
      const unsigned bal = __ballot_sync(0xffffffffu, pc == sh.pick && pc != a.halt);
      if (lane_id == 0) sh.warp_cnt[warp] = __popc(bal);
      __syncthreads();
      if (t == 0) {
        int c = 0;
        for (int w2 = 0; w2 < nwarps; ++w2) c += sh.warp_cnt[w2];
        sh.count = c;
      }
      __syncthreads();
    }
    const int b = sh.pick;
    if (b == a.halt) {  // every lane of this group halted and the queue is empty
      if (t == 0) a.group_done[g] = 1;
      break;
    }
    if (*(volatile int*)a.abort_flag) break;
    if (a.max_steps >= 0 && steps >= a.max_steps) {
      if (t == 0) {
        a.paused[0] = 1;
      }
      break;
    }
    if (a.trace_block != nullptr) {
      if (*a.trace_n >= a.trace_cap) {  // trace buffer full: pause, host drains and resumes
        if (t == 0) a.paused[1] = 1;
        break;
      }
    }

    // ---- execute block b for the lanes sitting at it
    const bool active = (pc == b);
    if (active && a.lane_trace != nullptr) {
      const long long c = *my_chain;
      const int n = a.lane_trace_len[c];
      if (n < a.lane_trace_cap) a.lane_trace[(size_t)c * a.lane_trace_cap + n] = b;
      a.lane_trace_len[c] = n + 1;
    }
    const ls_block blk = a.blocks[b];
    int my_fault = 0;  // 0 none, else op position + 1
    int fault_kind = 0, fault_var = 0, fault_detail = 0;
    for (int k = 0; k < blk.op_count; ++k) {
      const ls_op& op = a.ops[blk.op_begin + k];
      if (op.opcode == LS_OP_LEAPFROG) {  // cooperative superblock: every thread joins
        leapfrog_superblock(a.targets[op.imm0].P, a.targets[op.imm0].PT, a.targets[op.imm0].dim,
                            op, ln.ws, L, t, active && !my_fault, a.var_row, a.vars, lf_shared);
        continue;
      }
      if (!active || my_fault) continue;
      const int v = op.out;
      if (op.action == LS_POP) {
        int& s = ln.sp_of(v);
        if (s < 1) { my_fault = k + 1; fault_kind = LS_RUN_UNDERFLOW; fault_var = v; fault_detail = 0; continue; }
        --s;
        continue;
      }
      const ls_var& vd = a.vars[v];
      uint64_t* dst;
      if (vd.cls == LS_STACKED) {
        int& s = ln.sp_of(v);
        if (op.action == LS_PUSH) {
          if (s >= a.depth) { my_fault = k + 1; fault_kind = LS_RUN_OVERFLOW; fault_var = v; continue; }
          dst = ln.slot_ptr(v, s);
          compute_op(ln, op, dst);
          ++s;
          continue;
        }
        if (s < 1) { my_fault = k + 1; fault_kind = LS_RUN_UNDERFLOW; fault_var = v; fault_detail = 1; continue; }
        dst = ln.slot_ptr(v, s - 1);
      } else {
        dst = ln.slot_ptr(v, 0);
      }
      compute_op(ln, op, dst);
    }
    // ---- terminator
    bool halted_now = false;
    if (active && !my_fault) {
      int* top = &ln.pcs[(*pc_sp - 1) * L + t];
      switch (blk.term) {
        case LS_JUMP: *top = blk.a; break;
        case LS_BRANCH: *top = (ln.top(blk.cond)[0] != 0) ? blk.a : blk.b; break;
        case LS_PUSHJUMP:
          *top = blk.b;
          if (*pc_sp >= a.depth + 1) {
            my_fault = blk.op_count + 1; fault_kind = LS_RUN_OVERFLOW; fault_var = -1;
          } else {
            ln.pcs[(*pc_sp) * L + t] = blk.a;
            ++*pc_sp;
          }
          break;
        default:  // return
          if (*pc_sp < 1) {
            my_fault = blk.op_count + 1; fault_kind = LS_RUN_UNDERFLOW; fault_var = -1;
          } else {
            --*pc_sp;
            if (*pc_sp >= 1 && ln.pcs[(*pc_sp - 1) * L + t] == a.halt) halted_now = true;
          }
          break;
      }
    }
    if (my_fault) record_fault(a, &sh.fault_key, my_fault - 1, t);
    __syncthreads();
    if (sh.fault_key != ~0ull) {
      // the lowest (op position, lane) is the one the reference reports
      if ((unsigned)(sh.fault_key & 0xffffffffu) == (unsigned)t && my_fault &&
          (unsigned)(my_fault - 1) == (unsigned)(sh.fault_key >> 32)) {
        a.fault->key = sh.fault_key;
        a.fault->kind = fault_kind;
        a.fault->var = fault_var;
        a.fault->block = b;
        a.fault->detail = fault_detail;
        a.fault->chain = *my_chain;
        __threadfence();
        atomicExch(a.abort_flag, 1);
      }
      steps++;
      break;
    }
    if (halted_now) {
      write_output(a, ln, *my_chain);
      if (a.refill) *my_chain = -1;
    }
    // ---- bookkeeping: trace record, per-block totals, gradient counts
    if (t == 0) {
      if (a.trace_block != nullptr) {
        const long long n = *a.trace_n;
        a.trace_block[n] = b;
        a.trace_active[n] = sh.count;
        *a.trace_n = n + 1;
      }
      bsteps[b] += 1;
      bactive[b] += sh.count;
      useful += (unsigned long long)sh.count * (unsigned long long)blk.grads;
      launched += (unsigned long long)L * (unsigned long long)blk.grads;
    }
    ++steps;
    __syncthreads();
  }
  if (t == 0) {
    a.group_steps[g] = steps;
    if (useful) atomicAdd(a.useful, useful);
    if (launched) atomicAdd(a.launched, launched);
  }
}

// ---- small standalone kernels ----------------------------------------------------------

__global__ void rng_kernel(const int64_t* key, const int64_t* ctr, long long n, double* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = lsb::rng_uniform(key[i], ctr[i]);
}

__global__ void target_eval_kernel(DevTarget tg, int which, const double* x, long long z, double* out,
                                   uint64_t* scratch) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= z) return;
  // lane-minor copy so the per-lane primitives see their usual layout
  const int d = tg.dim;
  uint64_t* xs = scratch + i;  // stride z
  for (int j = 0; j < d; ++j) xs[(size_t)j * z] = f64_bits(x[(size_t)i * d + j]);
  if (which == 0) {
    out[i] = target_logpdf(tg, xs, (int)z, 1);
  } else {
    uint64_t* gs = scratch + (size_t)d * z + i;
    target_grad(tg, xs, (int)z, gs);
    for (int j = 0; j < d; ++j) out[(size_t)i * d + j] = as_f64(gs[(size_t)j * z]);
  }
}

}  // namespace

// =====================================================================================
// Host side: C ABI
// =====================================================================================

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) return fail(LS_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
static int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) return fail(LS_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return LS_OK;
}

struct ls_program {
  std::vector<ls_block> blocks;
  std::vector<ls_op> ops;
  std::vector<ls_var> vars;
  std::vector<int> inputs;
  int entry = 0, output = 0;
  int n_stacked = 0;
  int flat_rows = 0;
  ls_block* d_blocks = nullptr;
  ls_op* d_ops = nullptr;
  ls_var* d_vars = nullptr;
  int* d_inputs = nullptr;
  DevTarget targets[kMaxTargets];
  std::vector<double*> owned;
  int device = 0;
};

struct ls_machine {
  ls_program* p = nullptr;
  long long z = 0;
  int depth = 0, lanes = 0, groups = 0, group_rows = 0;
  ls_machine_opts opts{};
  std::vector<int> var_row, var_depth, input_width;
  int* d_var_row = nullptr;
  int* d_var_depth = nullptr;
  int* d_input_width = nullptr;
  uint64_t* ws = nullptr;
  int* sp = nullptr;
  int* pcs = nullptr;
  long long* chain_of = nullptr;
  std::vector<uint64_t*> inputs;
  uint64_t** d_input_ptrs = nullptr;
  uint64_t* output = nullptr;
  int out_width = 0;
  unsigned long long* counters = nullptr;  // [0] next_chain [1] useful [2] launched
  long long* group_steps = nullptr;
  int* group_done = nullptr;
  int* trace_block = nullptr;
  int* trace_active = nullptr;
  long long trace_cap = 0;
  long long* trace_n = nullptr;
  long long* blk_steps = nullptr;
  long long* blk_active = nullptr;
  FaultRec* fault = nullptr;
  int* flags = nullptr;  // [0] abort [1] paused-steps [2] paused-trace
  int* lane_trace = nullptr;
  int* lane_trace_len = nullptr;
  int lane_trace_cap = 0;
  bool started = false;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  long long launches = 0;
};

extern "C" {

int ls_abi_version(void) { return LS_ABI_VERSION; }

const char* ls_last_error(void) { return g_err.c_str(); }

int ls_device_count(int32_t* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *n = 0;
    return fail(LS_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  *n = c;
  return LS_OK;
}

int ls_program_create(const ls_program_desc* d, ls_program** out) {
  if (!d || !out || d->n_blocks < 1 || d->n_vars < 1) return fail(LS_EINVAL, "empty program");
  auto* p = new ls_program();
  p->blocks.assign(d->blocks, d->blocks + d->n_blocks);
  p->ops.assign(d->ops, d->ops + d->n_ops);
  p->vars.assign(d->vars, d->vars + d->n_vars);
  p->inputs.assign(d->inputs, d->inputs + d->n_inputs);
  p->entry = d->entry;
  p->output = d->output;
  p->flat_rows = d->flat_rows;
  for (auto& v : p->vars) if (v.cls == LS_STACKED) p->n_stacked = std::max(p->n_stacked, v.sp + 1);
  for (auto& b : p->blocks) {
    if (b.op_begin < 0 || b.op_begin + b.op_count > d->n_ops) { delete p; return fail(LS_EINVAL, "block op range"); }
  }
  cudaGetDevice(&p->device);
  int rc;
  if ((rc = dalloc(&p->d_blocks, p->blocks.size())) || (rc = dalloc(&p->d_ops, p->ops.size())) ||
      (rc = dalloc(&p->d_vars, p->vars.size())) || (rc = dalloc(&p->d_inputs, p->inputs.size()))) {
    ls_program_destroy(p);
    return rc;
  }
  cudaMemcpy(p->d_blocks, p->blocks.data(), p->blocks.size() * sizeof(ls_block), cudaMemcpyHostToDevice);
  if (!p->ops.empty()) cudaMemcpy(p->d_ops, p->ops.data(), p->ops.size() * sizeof(ls_op), cudaMemcpyHostToDevice);
  cudaMemcpy(p->d_vars, p->vars.data(), p->vars.size() * sizeof(ls_var), cudaMemcpyHostToDevice);
  if (!p->inputs.empty()) cudaMemcpy(p->d_inputs, p->inputs.data(), p->inputs.size() * sizeof(int), cudaMemcpyHostToDevice);
  CK(cudaGetLastError());
  *out = p;
  return LS_OK;
}

int ls_program_bind_target(ls_program* p, int32_t slot, int32_t kind, int32_t dim, int32_t n,
                           const double* params, double norm) {
  if (!p || slot < 0 || slot >= kMaxTargets || dim < 1) return fail(LS_EINVAL, "bad target slot");
  const int rows = kind == LS_TARGET_GAUSSIAN ? dim : n;
  if (rows < 1) return fail(LS_EINVAL, "bad target shape");
  std::vector<double> h(params, params + (size_t)rows * dim), ht((size_t)rows * dim);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < dim; ++j) ht[(size_t)j * rows + i] = h[(size_t)i * dim + j];
  double *dP = nullptr, *dPT = nullptr;
  int rc;
  if ((rc = dalloc(&dP, h.size())) || (rc = dalloc(&dPT, h.size()))) return rc;
  CK(cudaMemcpy(dP, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dPT, ht.data(), ht.size() * sizeof(double), cudaMemcpyHostToDevice));
  p->owned.push_back(dP);
  p->owned.push_back(dPT);
  p->targets[slot] = DevTarget{kind, dim, n, dP, dPT, norm};
  return LS_OK;
}

int ls_program_destroy(ls_program* p) {
  if (!p) return LS_OK;
  cudaFree(p->d_blocks);
  cudaFree(p->d_ops);
  cudaFree(p->d_vars);
  cudaFree(p->d_inputs);
  for (double* q : p->owned) cudaFree(q);
  delete p;
  return LS_OK;
}

int ls_machine_destroy(ls_machine* m) {
  if (!m) return LS_OK;
  if (m->stream) cudaStreamSynchronize(m->stream);
  cudaFree(m->d_var_row); cudaFree(m->d_var_depth); cudaFree(m->d_input_width);
  cudaFree(m->ws); cudaFree(m->sp); cudaFree(m->pcs); cudaFree(m->chain_of);
  for (auto* q : m->inputs) cudaFree(q);
  cudaFree(m->d_input_ptrs); cudaFree(m->output); cudaFree(m->counters);
  cudaFree(m->group_steps); cudaFree(m->group_done); cudaFree(m->trace_block);
  cudaFree(m->trace_active); cudaFree(m->trace_n); cudaFree(m->blk_steps);
  cudaFree(m->blk_active); cudaFree(m->fault); cudaFree(m->flags);
  cudaFree(m->lane_trace); cudaFree(m->lane_trace_len);
  if (m->ev0) cudaEventDestroy(m->ev0);
  if (m->ev1) cudaEventDestroy(m->ev1);
  if (m->stream) cudaStreamDestroy(m->stream);
  delete m;
  return LS_OK;
}

static int static_init(ls_machine* m);

int ls_machine_create(ls_program* p, int64_t z, int32_t depth, const ls_machine_opts* opts,
                      ls_machine** out) {
  if (!p || !out || z < 1 || depth < 1) return fail(LS_EINVAL, "bad machine arguments");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(LS_ECUDA, "no CUDA device: the lockstep B200 engine has no CPU fallback");
  }
  auto* m = new ls_machine();
  m->p = p;
  m->z = z;
  m->depth = depth;
  if (opts) m->opts = *opts;
  int lanes = m->opts.lanes_per_cta > 0 ? m->opts.lanes_per_cta : (int)std::min<long long>(z, kMaxLanes);
  if (m->opts.lanes_per_cta <= 0 && z > kMaxLanes) {
    delete m;
    return fail(LS_EINVAL, "a single schedule group holds at most 1024 lanes; set lanes_per_cta");
  }
  lanes = ((lanes + 31) / 32) * 32;
  if (lanes > kMaxLanes) lanes = kMaxLanes;
  m->lanes = lanes;
  const bool refill = z > lanes;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long want = (z + lanes - 1) / lanes;
  int groups = m->opts.ctas > 0 ? m->opts.ctas : sms * std::max(1, 1024 / lanes);
  if (!refill) groups = 1;
  if (groups > want) groups = (int)want;
  m->groups = groups;
  if (m->opts.trace && groups != 1) {
    delete m;
    return fail(LS_EINVAL, "per-step traces need a single schedule group (z <= lanes_per_cta)");
  }
  // workspace rows
  const auto& vars = p->vars;
  m->var_row.resize(vars.size());
  m->var_depth.resize(vars.size());
  int rows = p->flat_rows;  // non-stacked storage was laid out by the lowering
  for (size_t v = 0; v < vars.size(); ++v) {
    const int slots = vars[v].cls == LS_STACKED ? depth : 1;
    m->var_depth[v] = slots;
    if (vars[v].cls == LS_STACKED) {
      m->var_row[v] = rows;
      rows += slots * vars[v].width;
    } else {
      m->var_row[v] = vars[v].row;
      if (vars[v].row < 0 || vars[v].row + vars[v].width > p->flat_rows) {
        delete m;
        return fail(LS_EINVAL, "variable rows outside the flat region");
      }
    }
  }
  m->group_rows = rows;
  m->out_width = vars[p->output].width;
  for (int v : p->inputs) m->input_width.push_back(vars[v].width);
  const int n_sp_rows = p->n_stacked + 1;
  int rc = 0;
  CK(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
  const size_t L = lanes;
  if ((rc = dalloc(&m->d_var_row, vars.size())) || (rc = dalloc(&m->d_var_depth, vars.size())) ||
      (rc = dalloc(&m->d_input_width, std::max<size_t>(1, m->input_width.size()))) ||
      (rc = dalloc(&m->ws, (size_t)groups * rows * L)) ||
      (rc = dalloc(&m->sp, (size_t)groups * n_sp_rows * L)) ||
      (rc = dalloc(&m->pcs, (size_t)groups * (depth + 1) * L)) ||
      (rc = dalloc(&m->chain_of, (size_t)groups * L)) ||
      (rc = dalloc(&m->d_input_ptrs, std::max<size_t>(1, p->inputs.size()))) ||
      (rc = dalloc(&m->output, (size_t)z * m->out_width)) ||
      (rc = dalloc(&m->counters, 4)) || (rc = dalloc(&m->group_steps, groups)) ||
      (rc = dalloc(&m->group_done, groups)) ||
      (rc = dalloc(&m->blk_steps, (size_t)groups * p->blocks.size())) ||
      (rc = dalloc(&m->blk_active, (size_t)groups * p->blocks.size())) ||
      (rc = dalloc(&m->fault, 1)) || (rc = dalloc(&m->flags, 4)) || (rc = dalloc(&m->trace_n, 1))) {
    ls_machine_destroy(m);
    return rc;
  }
  for (size_t k = 0; k < p->inputs.size(); ++k) {
    uint64_t* buf = nullptr;
    if ((rc = dalloc(&buf, (size_t)z * m->input_width[k]))) { ls_machine_destroy(m); return rc; }
    m->inputs.push_back(buf);
  }
  cudaMemcpy(m->d_var_row, m->var_row.data(), vars.size() * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(m->d_var_depth, m->var_depth.data(), vars.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (!m->input_width.empty())
    cudaMemcpy(m->d_input_width, m->input_width.data(), m->input_width.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (!m->inputs.empty())
    cudaMemcpy(m->d_input_ptrs, m->inputs.data(), m->inputs.size() * sizeof(uint64_t*), cudaMemcpyHostToDevice);
  // the reference zero-fills all storage at init (pc_vm.py:171-181)
  cudaMemsetAsync(m->ws, 0, (size_t)groups * rows * L * sizeof(uint64_t), m->stream);
  cudaMemsetAsync(m->sp, 0, (size_t)groups * n_sp_rows * L * sizeof(int), m->stream);
  cudaMemsetAsync(m->pcs, 0, (size_t)groups * (depth + 1) * L * sizeof(int), m->stream);
  cudaMemsetAsync(m->output, 0, (size_t)z * m->out_width * sizeof(uint64_t), m->stream);
  cudaMemsetAsync(m->counters, 0, 4 * sizeof(unsigned long long), m->stream);
  cudaMemsetAsync(m->group_steps, 0, groups * sizeof(long long), m->stream);
  cudaMemsetAsync(m->group_done, 0, groups * sizeof(int), m->stream);
  cudaMemsetAsync(m->blk_steps, 0, (size_t)groups * p->blocks.size() * sizeof(long long), m->stream);
  cudaMemsetAsync(m->blk_active, 0, (size_t)groups * p->blocks.size() * sizeof(long long), m->stream);
  cudaMemsetAsync(m->flags, 0, 4 * sizeof(int), m->stream);
  cudaMemsetAsync(m->trace_n, 0, sizeof(long long), m->stream);
  FaultRec f0{~0ull, 0, 0, 0, 0, -1};
  cudaMemcpyAsync(m->fault, &f0, sizeof(f0), cudaMemcpyHostToDevice, m->stream);
  // chain slots: static assignment for a single group, else -1 (free, refill)
  std::vector<long long> slots((size_t)groups * L, -1);
  if (!refill) {
    for (size_t t = 0; t < L; ++t) slots[t] = (long long)t < z ? (long long)t : -2;
  }
  cudaMemcpyAsync(m->chain_of, slots.data(), slots.size() * sizeof(long long), cudaMemcpyHostToDevice, m->stream);
  if (m->opts.lane_trace_cap > 0) {  // per-chain pc traces
    m->lane_trace_cap = m->opts.lane_trace_cap;
    if ((rc = dalloc(&m->lane_trace, (size_t)z * m->lane_trace_cap)) ||
        (rc = dalloc(&m->lane_trace_len, (size_t)z))) {
      ls_machine_destroy(m);
      return rc;
    }
    cudaMemsetAsync(m->lane_trace_len, 0, (size_t)z * sizeof(int), m->stream);
  }
  if (m->opts.trace) {
    m->trace_cap = 1 << 16;
    if ((rc = dalloc(&m->trace_block, m->trace_cap)) || (rc = dalloc(&m->trace_active, m->trace_cap))) {
      ls_machine_destroy(m);
      return rc;
    }
  }
  CK(cudaStreamSynchronize(m->stream));
  CK(cudaGetLastError());
  if ((rc = static_init(m))) {
    ls_machine_destroy(m);
    return rc;
  }
  *out = m;
  return LS_OK;
}

int ls_machine_reset(ls_machine* m) {
  if (!m) return fail(LS_EINVAL, "null machine");
  const size_t L = m->lanes, nb = m->p->blocks.size();
  const int n_sp_rows = m->p->n_stacked + 1;
  CK(cudaMemsetAsync(m->sp, 0, (size_t)m->groups * n_sp_rows * L * sizeof(int), m->stream));
  CK(cudaMemsetAsync(m->pcs, 0, (size_t)m->groups * (m->depth + 1) * L * sizeof(int), m->stream));
  CK(cudaMemsetAsync(m->counters, 0, 4 * sizeof(unsigned long long), m->stream));
  CK(cudaMemsetAsync(m->group_steps, 0, m->groups * sizeof(long long), m->stream));
  CK(cudaMemsetAsync(m->group_done, 0, m->groups * sizeof(int), m->stream));
  CK(cudaMemsetAsync(m->blk_steps, 0, (size_t)m->groups * nb * sizeof(long long), m->stream));
  CK(cudaMemsetAsync(m->blk_active, 0, (size_t)m->groups * nb * sizeof(long long), m->stream));
  CK(cudaMemsetAsync(m->flags, 0, 4 * sizeof(int), m->stream));
  CK(cudaMemsetAsync(m->trace_n, 0, sizeof(long long), m->stream));
  if (m->lane_trace_len) CK(cudaMemsetAsync(m->lane_trace_len, 0, (size_t)m->z * sizeof(int), m->stream));
  FaultRec f0{~0ull, 0, 0, 0, 0, -1};
  CK(cudaMemcpyAsync(m->fault, &f0, sizeof(f0), cudaMemcpyHostToDevice, m->stream));
  const bool refill = m->z > m->lanes;
  std::vector<long long> slots((size_t)m->groups * L, -1);
  if (!refill)
    for (size_t t = 0; t < L; ++t) slots[t] = (long long)t < m->z ? (long long)t : -2;
  CK(cudaMemcpyAsync(m->chain_of, slots.data(), slots.size() * sizeof(long long), cudaMemcpyHostToDevice, m->stream));
  CK(cudaStreamSynchronize(m->stream));
  m->started = false;
  return static_init(m);
}

int ls_machine_set_input(ls_machine* m, int32_t idx, const void* host, int64_t bytes) {
  if (!m || idx < 0 || idx >= (int)m->inputs.size()) return fail(LS_EINVAL, "bad input index");
  const int64_t want = m->z * m->input_width[idx] * 8;
  if (bytes != want) return fail(LS_EINVAL, "input size mismatch");
  CK(cudaMemcpyAsync(m->inputs[idx], host, bytes, cudaMemcpyHostToDevice, m->stream));
  CK(cudaStreamSynchronize(m->stream));
  return static_init(m);
}

int ls_machine_set_input_device(ls_machine* m, int32_t idx, const void* dev, int64_t bytes) {
  if (!m || idx < 0 || idx >= (int)m->inputs.size()) return fail(LS_EINVAL, "bad input index");
  const int64_t want = m->z * m->input_width[idx] * 8;
  if (bytes != want) return fail(LS_EINVAL, "input size mismatch");
  CK(cudaMemcpyAsync(m->inputs[idx], dev, bytes, cudaMemcpyDeviceToDevice, m->stream));
  return static_init(m);
}

__global__ void init_static_kernel(const __grid_constant__ VMArgs a) {
  const int t = threadIdx.x;
  const long long c = a.chain_of[t];
  if (c < 0) return;
  Lane ln{&a, a.ws, a.sp, a.pcs, t, a.lanes};
  init_lane(a, ln, c);
}

static VMArgs make_args(ls_machine* m, long long max_steps) {
  ls_program* p = m->p;
  VMArgs a{};
  a.blocks = p->d_blocks; a.ops = p->d_ops; a.vars = p->d_vars;
  a.var_row = m->d_var_row; a.var_depth = m->d_var_depth;
  a.n_blocks = (int)p->blocks.size(); a.halt = (int)p->blocks.size(); a.entry = p->entry;
  a.n_inputs = (int)p->inputs.size(); a.input_vars = p->d_inputs; a.output_var = p->output;
  a.n_sp_rows = p->n_stacked + 1;
  for (int i = 0; i < kMaxTargets; ++i) a.targets[i] = p->targets[i];
  a.z = m->z; a.depth = m->depth; a.lanes = m->lanes; a.group_rows = m->group_rows;
  a.ws = m->ws; a.sp = m->sp; a.pcs = m->pcs; a.chain_of = m->chain_of;
  a.inputs = (const uint64_t* const*)m->d_input_ptrs; a.input_width = m->d_input_width;
  a.output = m->output; a.out_width = m->out_width;
  a.next_chain = m->counters + 0;
  a.refill = m->groups > 1 || m->z > m->lanes;
  a.sched = m->opts.sched;
  a.exact_logpdf = m->opts.exact_logpdf;
  a.max_steps = max_steps;
  a.group_steps = m->group_steps; a.group_done = m->group_done;
  a.trace_block = m->trace_block; a.trace_active = m->trace_active;
  a.trace_cap = m->trace_cap; a.trace_n = m->trace_n;
  a.blk_steps = m->blk_steps; a.blk_active = m->blk_active;
  a.useful = m->counters + 1; a.launched = m->counters + 2;
  a.fault = m->fault; a.abort_flag = m->flags + 0; a.paused = m->flags + 1;
  a.lane_trace = m->lane_trace; a.lane_trace_len = m->lane_trace_len;
  a.lane_trace_cap = m->lane_trace_cap;
  return a;
}

// Single-group machines are seeded eagerly (pc stack [halt, entry], one live
// slot per data stack, inputs in slot 0) so observers can inspect them before
// the first step; refilling machines seed each lane when it takes a chain.
static int static_init(ls_machine* m) {
  VMArgs a = make_args(m, 0);
  if (a.refill || m->started) return LS_OK;
  init_static_kernel<<<1, m->lanes, 0, m->stream>>>(a);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(m->stream));
  return LS_OK;
}

int ls_run(ls_machine* m, int64_t max_steps, ls_status* st) {
  if (!m || !st) return fail(LS_EINVAL, "null machine");
  ls_program* p = m->p;
  VMArgs a = make_args(m, max_steps);
  m->started = true;
  const size_t smem = (p->blocks.size() + 1) * sizeof(int);
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(vm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaMemsetAsync(m->flags + 1, 0, 2 * sizeof(int), m->stream));
  if (!m->ev0) {
    CK(cudaEventCreate(&m->ev0));
    CK(cudaEventCreate(&m->ev1));
  }
  CK(cudaEventRecord(m->ev0, m->stream));
  vm_kernel<<<m->groups, m->lanes, smem, m->stream>>>(a);
  CK(cudaGetLastError());
  CK(cudaEventRecord(m->ev1, m->stream));
  CK(cudaStreamSynchronize(m->stream));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
  m->launches += 1;
  int flags[3];
  FaultRec f;
  std::vector<long long> gsteps(m->groups);
  std::vector<int> gdone(m->groups);
  unsigned long long cnt[3];
  CK(cudaMemcpy(flags, m->flags, sizeof(flags), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&f, m->fault, sizeof(f), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(gsteps.data(), m->group_steps, m->groups * sizeof(long long), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(gdone.data(), m->group_done, m->groups * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cnt, m->counters, sizeof(cnt), cudaMemcpyDeviceToHost));
  std::memset(st, 0, sizeof(*st));
  st->steps = *std::max_element(gsteps.begin(), gsteps.end());
  st->kernel_ms = ms;
  st->launches = m->launches;
  st->useful_grads = (int64_t)cnt[1];
  st->launched_grads = (int64_t)cnt[2];
  st->var = -1;
  if (flags[0]) {
    st->kind = f.kind;
    st->var = f.var;
    st->lane = f.chain;
    st->block = f.block;
    st->pad = f.detail;
    return LS_OK;
  }
  bool all_done = true;
  for (int d : gdone) all_done = all_done && d;
  if (all_done) st->kind = LS_RUN_HALTED;
  else if (flags[1] && max_steps >= 0 && st->steps >= max_steps) st->kind = LS_RUN_STEP_LIMIT;
  else st->kind = LS_RUN_PAUSED;
  return LS_OK;
}

int ls_read_output(ls_machine* m, void* host, int64_t bytes) {
  if (!m) return fail(LS_EINVAL, "null machine");
  if (bytes != m->z * m->out_width * 8) return fail(LS_EINVAL, "output size mismatch");
  CK(cudaMemcpyAsync(host, m->output, bytes, cudaMemcpyDeviceToHost, m->stream));
  CK(cudaStreamSynchronize(m->stream));
  return LS_OK;
}

int ls_output_device(ls_machine* m, void** dev) {
  if (!m || !dev) return fail(LS_EINVAL, "null machine");
  *dev = m->output;
  return LS_OK;
}

int ls_trace_fetch(ls_machine* m, int32_t* blocks, int32_t* active, int64_t cap, int64_t* n) {
  if (!m || !n) return fail(LS_EINVAL, "null machine");
  *n = 0;
  if (!m->trace_block) return LS_OK;
  long long have = 0;
  CK(cudaMemcpy(&have, m->trace_n, sizeof(have), cudaMemcpyDeviceToHost));
  const long long k = std::min<long long>(have, cap);
  if (k > 0) {
    CK(cudaMemcpy(blocks, m->trace_block, k * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(active, m->trace_active, k * sizeof(int), cudaMemcpyDeviceToHost));
  }
  // drain: shift any remainder (cap < have) to the front
  if (k < have) {
    std::vector<int> rb(have - k), ra(have - k);
    CK(cudaMemcpy(rb.data(), m->trace_block + k, (have - k) * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ra.data(), m->trace_active + k, (have - k) * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(m->trace_block, rb.data(), rb.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(m->trace_active, ra.data(), ra.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  const long long rest = have - k;
  CK(cudaMemcpy(m->trace_n, &rest, sizeof(rest), cudaMemcpyHostToDevice));
  *n = k;
  return LS_OK;
}

int ls_block_totals(ls_machine* m, int64_t* steps, int64_t* active) {
  if (!m) return fail(LS_EINVAL, "null machine");
  const size_t nb = m->p->blocks.size();
  std::vector<long long> s((size_t)m->groups * nb), a((size_t)m->groups * nb);
  CK(cudaMemcpy(s.data(), m->blk_steps, s.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(a.data(), m->blk_active, a.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  for (size_t b = 0; b < nb; ++b) {
    long long ss = 0, aa = 0;
    for (int g = 0; g < m->groups; ++g) { ss += s[(size_t)g * nb + b]; aa += a[(size_t)g * nb + b]; }
    steps[b] = ss;
    active[b] = aa;
  }
  return LS_OK;
}

int ls_read_var(ls_machine* m, int32_t var, void* host, int64_t bytes) {
  if (!m || var < 0 || var >= (int)m->p->vars.size()) return fail(LS_EINVAL, "bad var");
  if (m->groups != 1) return fail(LS_EINVAL, "observer access needs a single schedule group");
  const int slots = m->var_depth[var], w = m->p->vars[var].width;
  const long long z = m->z;
  if (bytes != (int64_t)slots * z * w * 8) return fail(LS_EINVAL, "var size mismatch");
  std::vector<uint64_t> raw((size_t)slots * w * m->lanes);
  CK(cudaMemcpy(raw.data(), m->ws + (size_t)m->var_row[var] * m->lanes, raw.size() * 8, cudaMemcpyDeviceToHost));
  auto* dst = static_cast<uint64_t*>(host);
  for (int s = 0; s < slots; ++s)
    for (long long l = 0; l < z; ++l)
      for (int i = 0; i < w; ++i)
        dst[((size_t)s * z + l) * w + i] = raw[((size_t)s * w + i) * m->lanes + l];
  return LS_OK;
}

int ls_read_pointers(ls_machine* m, int32_t var, int64_t* host, int64_t z) {
  if (!m || z != m->z) return fail(LS_EINVAL, "bad pointer request");
  if (m->groups != 1) return fail(LS_EINVAL, "observer access needs a single schedule group");
  int row;
  if (var < 0) row = m->p->n_stacked;
  else if (m->p->vars[var].cls == LS_STACKED) row = m->p->vars[var].sp;
  else return fail(LS_EINVAL, "not a stacked variable");
  std::vector<int> raw(m->lanes);
  CK(cudaMemcpy(raw.data(), m->sp + (size_t)row * m->lanes, m->lanes * sizeof(int), cudaMemcpyDeviceToHost));
  for (long long l = 0; l < z; ++l) host[l] = raw[l];
  return LS_OK;
}

int ls_read_pc_stack(ls_machine* m, int32_t* host, int64_t count) {
  if (!m || count != (int64_t)(m->depth + 1) * m->z) return fail(LS_EINVAL, "bad pc request");
  std::vector<int> raw((size_t)(m->depth + 1) * m->lanes);
  CK(cudaMemcpy(raw.data(), m->pcs, raw.size() * sizeof(int), cudaMemcpyDeviceToHost));
  for (int s = 0; s <= m->depth; ++s)
    for (long long l = 0; l < m->z; ++l) host[(size_t)s * m->z + l] = raw[(size_t)s * m->lanes + l];
  return LS_OK;
}

int ls_lane_trace_fetch(ls_machine* m, int32_t* blocks, int32_t* lens, int64_t cap) {
  if (!m || !m->lane_trace) return fail(LS_EINVAL, "machine was created without lane traces");
  if (cap != m->lane_trace_cap) return fail(LS_EINVAL, "lane trace capacity mismatch");
  CK(cudaMemcpy(blocks, m->lane_trace, (size_t)m->z * cap * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(lens, m->lane_trace_len, (size_t)m->z * sizeof(int), cudaMemcpyDeviceToHost));
  return LS_OK;
}

int ls_machine_sync(ls_machine* m) {
  if (!m) return fail(LS_EINVAL, "null machine");
  CK(cudaStreamSynchronize(m->stream));
  return LS_OK;
}

int ls_rng_uniform(const int64_t* key, const int64_t* counter, int64_t n, double* out) {
  if (n <= 0) return LS_OK;
  int64_t *dk = nullptr, *dc = nullptr;
  double* dout = nullptr;
  int rc;
  if ((rc = dalloc(&dk, n)) || (rc = dalloc(&dc, n)) || (rc = dalloc(&dout, n))) {
    cudaFree(dk); cudaFree(dc);
    return rc;
  }
  cudaMemcpy(dk, key, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, counter, n * 8, cudaMemcpyHostToDevice);
  rng_kernel<<<(unsigned)((n + 255) / 256), 256>>>(dk, dc, n, dout);
  cudaError_t e = cudaMemcpy(out, dout, n * 8, cudaMemcpyDeviceToHost);
  cudaFree(dk); cudaFree(dc); cudaFree(dout);
  if (e != cudaSuccess) return fail(LS_ECUDA, cudaGetErrorString(e));
  return LS_OK;
}

int ls_target_eval(int32_t kind, int32_t which, int32_t dim, int32_t n, const double* params,
                   double norm, const double* x, int64_t z, double* out) {
  if (z <= 0) return LS_OK;
  ls_program tmp;
  int rc = ls_program_bind_target(&tmp, 0, kind, dim, n, params, norm);
  if (rc) return rc;
  double *dx = nullptr, *dout = nullptr;
  uint64_t* scratch = nullptr;
  const size_t outn = which == 0 ? (size_t)z : (size_t)z * dim;
  if ((rc = dalloc(&dx, (size_t)z * dim)) || (rc = dalloc(&dout, outn)) ||
      (rc = dalloc(&scratch, (size_t)2 * z * dim))) {
    cudaFree(dx); cudaFree(dout);
    for (double* q : tmp.owned) cudaFree(q);
    tmp.owned.clear();
    return rc;
  }
  cudaMemcpy(dx, x, (size_t)z * dim * 8, cudaMemcpyHostToDevice);
  target_eval_kernel<<<(unsigned)((z + 127) / 128), 128>>>(tmp.targets[0], which, dx, z, dout, scratch);
  cudaError_t e = cudaMemcpy(out, dout, outn * 8, cudaMemcpyDeviceToHost);
  cudaFree(dx); cudaFree(dout); cudaFree(scratch);
  for (double* q : tmp.owned) cudaFree(q);
  tmp.owned.clear();
  if (e != cudaSuccess) return fail(LS_ECUDA, cudaGetErrorString(e));
  return LS_OK;
}

}  // extern "C"
