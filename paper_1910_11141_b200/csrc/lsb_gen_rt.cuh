// lsb_gen_rt.cuh — runtime helpers for generated (program-specialised) block code.
//
// codegen.py turns every flat block of a lowered program into straight-line
// CUDA (the paper's "static block / dynamic pc" partial evaluation,
// arXiv 1910.11141 §5): operand rows and widths become constants, block-local
// scalars live in registers, and only vectors, registers and stacks touch the
// lane-minor workspace. These helpers are the vector kernels it calls, with
// the same arithmetic as lsb_vm.cuh::compute_op (warp engine: stride 32).
#pragma once
#include <cstdint>

#include "lsb_vm.cuh"

namespace lsbgen {

using lsb::as_f64;
using lsb::f64_bits;
using namespace lsbvm;

constexpr int S = 32;  // lane stride of the warp engine

#ifndef LSB_EW_UNROLL
#define LSB_EW_UNROLL 16
#endif
constexpr int kEw = LSB_EW_UNROLL;

// dst[i] = f(i) for i < W, kEw loads in flight before the stores
template <int W, class F>
__device__ __forceinline__ void ew(uint64_t* dst, const F& f) {
  constexpr int full = W / kEw * kEw;
#pragma unroll 1
  for (int i = 0; i < full; i += kEw) {
    uint64_t v[kEw];
#pragma unroll
    for (int j = 0; j < kEw; ++j) v[j] = f(i + j);
#pragma unroll
    for (int j = 0; j < kEw; ++j) dst[(i + j) * S] = v[j];
  }
#pragma unroll
  for (int i = full; i < W; ++i) dst[i * S] = f(i);
}

#ifndef LSB_GEN_OOL
#define LSB_GEN_OOL 0
#endif

// Runtime-width form of ew for the shared out-of-line helpers below: kEw loads in
// flight per batch, the tail as one predicated batch.
template <class F>
__device__ __forceinline__ void ew_n(uint64_t* dst, int w, const F& f) {
#pragma unroll 1
  for (int i = 0; i < w; i += kEw) {
    uint64_t v[kEw];
    if (i + kEw <= w) {
#pragma unroll
      for (int j = 0; j < kEw; ++j) v[j] = f(i + j);
#pragma unroll
      for (int j = 0; j < kEw; ++j) dst[(i + j) * S] = v[j];
    } else {
#pragma unroll
      for (int j = 0; j < kEw; ++j)
        if (i + j < w) v[j] = f(i + j);
#pragma unroll
      for (int j = 0; j < kEw; ++j)
        if (i + j < w) dst[(i + j) * S] = v[j];
    }
  }
}

// Out-of-line vector helpers (LSB_GEN_OOL): every block calls one shared body
// instead of inlining a loop per call site, which keeps the generated program's
// instruction footprint small enough for the SM instruction caches.
__device__ __noinline__ void copy_n(uint64_t* dst, const uint64_t* src, int w) {
  if (dst != src) ew_n(dst, w, [&](int i) { return src[i * S]; });
}
__device__ __noinline__ void fill_n(uint64_t* dst, uint64_t v, int w) {
  ew_n(dst, w, [&](int) { return v; });
}
__device__ __noinline__ void axpy_n(uint64_t* dst, double s, const uint64_t* x, const uint64_t* y, int w) {
  ew_n(dst, w, [&](int i) { return f64_bits(__dadd_rn(__dmul_rn(s, as_f64(x[i * S])), as_f64(y[i * S]))); });
}
// f64 add / sub / mul / div (op 0..3), IEEE round-to-nearest like compute_op
__device__ __noinline__ void binop_f64_n(uint64_t* dst, const uint64_t* x, const uint64_t* y, int w, int op) {
  switch (op) {
    case 0: ew_n(dst, w, [&](int i) { return f64_bits(__dadd_rn(as_f64(x[i * S]), as_f64(y[i * S]))); }); break;
    case 1: ew_n(dst, w, [&](int i) { return f64_bits(__dsub_rn(as_f64(x[i * S]), as_f64(y[i * S]))); }); break;
    case 2: ew_n(dst, w, [&](int i) { return f64_bits(__dmul_rn(as_f64(x[i * S]), as_f64(y[i * S]))); }); break;
    default: ew_n(dst, w, [&](int i) { return f64_bits(__ddiv_rn(as_f64(x[i * S]), as_f64(y[i * S]))); }); break;
  }
}
__device__ __noinline__ uint64_t ool_rng(int64_t key, int64_t c) { return f64_bits(lsb::rng_uniform(key, c)); }

template <int W>
__device__ __forceinline__ void copy(uint64_t* dst, const uint64_t* src) {
#if LSB_GEN_OOL
  copy_n(dst, src, W);
#else
  if (dst != src) ew<W>(dst, [&](int i) { return src[i * S]; });
#endif
}

// Copy between rows the generator proved disjoint, software-pipelined: the loads of
// batch k+1 are issued before the stores of batch k, so two batches (2 kEw words per
// thread) are in flight instead of one round trip per batch. Only valid without
// overlap — the loads run ahead of the stores.
template <int W>
__device__ __forceinline__ void copy_nr(uint64_t* __restrict__ dst, const uint64_t* __restrict__ src) {
  constexpr int full = W / kEw * kEw;
  if constexpr (full >= 2 * kEw) {
    uint64_t v[kEw];
#pragma unroll
    for (int j = 0; j < kEw; ++j) v[j] = src[j * S];
#pragma unroll 1
    for (int i = kEw; i < full; i += kEw) {
      uint64_t u[kEw];
#pragma unroll
      for (int j = 0; j < kEw; ++j) u[j] = src[(i + j) * S];
#pragma unroll
      for (int j = 0; j < kEw; ++j) dst[(i - kEw + j) * S] = v[j];
#pragma unroll
      for (int j = 0; j < kEw; ++j) v[j] = u[j];
    }
    if constexpr (full < W) {  // tail loads join the last batch's stores
      uint64_t t[W - full];
#pragma unroll
      for (int j = 0; j < W - full; ++j) t[j] = src[(full + j) * S];
#pragma unroll
      for (int j = 0; j < kEw; ++j) dst[(full - kEw + j) * S] = v[j];
#pragma unroll
      for (int j = 0; j < W - full; ++j) dst[(full + j) * S] = t[j];
    } else {
#pragma unroll
      for (int j = 0; j < kEw; ++j) dst[(full - kEw + j) * S] = v[j];
    }
  } else {
    ew<W>(dst, [&](int i) { return src[i * S]; });
  }
}

// Long copies through the warp's shared-memory staging area with cp.async
// (LDGSTS): every thread issues all loads of a chunk for its own lane without
// holding registers, waits once, then stores — one memory round trip per
// chunk of CHUNK rows instead of one per 8 rows. Each thread only touches its
// own lane's column of the staging area, so no warp synchronisation is needed.
constexpr int kStageRows = 48;  // 48 rows x 32 lanes x 8 B = 12 KB per warp
using lsb::cp_async8;
using lsb::cp_async_wait_all;

template <int W>
__device__ __forceinline__ void copy_staged(uint64_t* dst, const uint64_t* src, double* sm) {
  if (dst == src) return;
  const int lane = threadIdx.x & 31;
  uint64_t* stage = reinterpret_cast<uint64_t*>(sm) + lane;
#pragma unroll 1
  for (int c0 = 0; c0 < W; c0 += kStageRows) {
    const int n = W - c0 < kStageRows ? W - c0 : kStageRows;
    for (int i = 0; i < n; ++i) cp_async8(stage + i * S, src + (c0 + i) * S);
    cp_async_wait_all();
    for (int i = 0; i < n; ++i) dst[(c0 + i) * S] = stage[i * S];
  }
}

// out-of-line libdevice transcendentals (same results as the inline calls)
__device__ __noinline__ double ool_exp(double x) { return exp(x); }
__device__ __noinline__ double ool_log(double x) { return log(x); }
__device__ __noinline__ double ool_sin(double x) { return sin(x); }
__device__ __noinline__ double ool_cos(double x) { return cos(x); }

// One source vector copied to N destinations (codegen fan-out of copies that share a
// source): each element is loaded once and stored N times, kEw loads in flight.
template <int W, int N>
__device__ __forceinline__ void copy_fan(const uint64_t* src, uint64_t* const (&dst)[N]) {
  constexpr int full = W / kEw * kEw;
#pragma unroll 1
  for (int i = 0; i < full; i += kEw) {
    uint64_t v[kEw];
#pragma unroll
    for (int j = 0; j < kEw; ++j) v[j] = src[(i + j) * S];
#pragma unroll
    for (int n = 0; n < N; ++n)
#pragma unroll
      for (int j = 0; j < kEw; ++j) dst[n][(i + j) * S] = v[j];
  }
  if constexpr (full < W) {
    uint64_t v[W - full];
#pragma unroll
    for (int j = 0; j < W - full; ++j) v[j] = src[(full + j) * S];
#pragma unroll
    for (int n = 0; n < N; ++n)
#pragma unroll
      for (int j = 0; j < W - full; ++j) dst[n][(full + j) * S] = v[j];
  }
}

template <int W>
__device__ __forceinline__ void fill(uint64_t* dst, uint64_t v) {
#if LSB_GEN_OOL
  if constexpr (W > 4) { fill_n(dst, v, W); return; }
#endif
  ew<W>(dst, [&](int) { return v; });
}

template <int W>
__device__ __forceinline__ void axpy(uint64_t* dst, double s, const uint64_t* x, const uint64_t* y) {
#if LSB_GEN_OOL
  axpy_n(dst, s, x, y, W);
#else
  ew<W>(dst, [&](int i) { return f64_bits(__dadd_rn(__dmul_rn(s, as_f64(x[i * S])), as_f64(y[i * S]))); });
#endif
}

template <int W>
__device__ __forceinline__ void select(uint64_t* dst, bool c, const uint64_t* x, const uint64_t* y) {
  const uint64_t* src = c ? x : y;
#if LSB_GEN_OOL
  copy_n(dst, src, W);
#else
  if (src != dst) ew<W>(dst, [&](int i) { return src[i * S]; });
#endif
}

// (x OP y).a and (x OP y).b (OP 0 = add, 1 = sub; TWO = second dot) for 8 <= W <= 128 without
// storing x OP y: every element, product and partial sum rounds exactly as the separate
// `t = x OP y; dot(t, a); dot(t, b)` ops (dot<W>'s numpy pairwise order), in one pass.
template <int W, int OP, bool TWO>
__device__ __forceinline__ void ew_dot(const uint64_t* x, const uint64_t* y, const uint64_t* a,
                                       const uint64_t* b, double& ra, double& rb) {
  static_assert(W >= 8 && W <= 128, "pairwise block form");
  auto t = [&](int i) {
    const double xv = as_f64(x[i * S]), yv = as_f64(y[i * S]);
    return OP == 0 ? __dadd_rn(xv, yv) : __dsub_rn(xv, yv);
  };
  constexpr int stop = W - W % 8;
  double r1[8], r2[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double tv = t(j);
    r1[j] = __dmul_rn(tv, as_f64(a[j * S]));
    if (TWO) r2[j] = __dmul_rn(tv, as_f64(b[j * S]));
  }
#pragma unroll 1  // one 8-element block (up to 32 loads) per iteration: no spills
  for (int i = 8; i < stop; i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double tv = t(i + j);
      r1[j] = __dadd_rn(r1[j], __dmul_rn(tv, as_f64(a[(i + j) * S])));
      if (TWO) r2[j] = __dadd_rn(r2[j], __dmul_rn(tv, as_f64(b[(i + j) * S])));
    }
  double s1 = __dadd_rn(__dadd_rn(__dadd_rn(r1[0], r1[1]), __dadd_rn(r1[2], r1[3])),
                        __dadd_rn(__dadd_rn(r1[4], r1[5]), __dadd_rn(r1[6], r1[7])));
  double s2 = 0.0;
  if (TWO)
    s2 = __dadd_rn(__dadd_rn(__dadd_rn(r2[0], r2[1]), __dadd_rn(r2[2], r2[3])),
                   __dadd_rn(__dadd_rn(r2[4], r2[5]), __dadd_rn(r2[6], r2[7])));
#pragma unroll
  for (int i = stop; i < W; ++i) {
    const double tv = t(i);
    s1 = __dadd_rn(s1, __dmul_rn(tv, as_f64(a[i * S])));
    if (TWO) s2 = __dadd_rn(s2, __dmul_rn(tv, as_f64(b[i * S])));
  }
  ra = __dadd_rn(0.0, s1);
  rb = __dadd_rn(0.0, s2);
}

// Shared out-of-line (x*y).sum() for 8 <= w <= 128 in numpy's pairwise order,
// 16 products loaded per batch.
__device__ __noinline__ double dot_n(const uint64_t* x, const uint64_t* y, int w) {
  auto p = [&](int i) { return __dmul_rn(as_f64(x[i * S]), as_f64(y[i * S])); };
  const int stop = w - w % 8;
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = p(j);
#pragma unroll 1
  for (int i = 8; i < stop; i += 16) {
    double v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = (i + j < stop) ? p(i + j) : 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v[j]);
    if (i + 8 < stop) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v[8 + j]);
    }
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (int i = stop; i < w; ++i) res = __dadd_rn(res, p(i));
  return __dadd_rn(0.0, res);
}

// (x*y).sum(): numpy's pairwise order (lsb_ops.cuh pairwise); for 8 <= W <= 128 the
// 8-accumulator block form with 16 products loaded per batch (a full unroll would
// hoist all 2W loads and spill).
template <int W>
__device__ __forceinline__ double dot(const uint64_t* x, const uint64_t* y) {
#if LSB_GEN_OOL
  if constexpr (W >= 8 && W <= 128) return dot_n(x, y, W);
#endif
  if constexpr (W < 8 || W > 128) {
    return lsb::dot_lane(x, y, W, S);
  } else {
    auto p = [&](int i) { return __dmul_rn(as_f64(x[i * S]), as_f64(y[i * S])); };
    constexpr int stop = W - W % 8;
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = p(j);
#pragma unroll 1
    for (int i = 8; i < stop; i += 16) {
      double v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = (i + j < stop) ? p(i + j) : 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v[j]);
      if (i + 8 < stop) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v[8 + j]);
      }
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
    for (int i = stop; i < W; ++i) res = __dadd_rn(res, p(i));
    return __dadd_rn(0.0, res);
  }
}

__device__ __forceinline__ int64_t to_i64(uint64_t w, bool is_f64) {
  return is_f64 ? lsb::f64_to_i64(as_f64(w)) : (int64_t)w;
}

__device__ __forceinline__ int64_t clip(int64_t k, int w) { return k < 0 ? 0 : (k > w - 1 ? w - 1 : k); }

__device__ __forceinline__ uint64_t i64_div(uint64_t a, uint64_t b) {  // numpy floor_divide, /0 -> 0
  const int64_t p = (int64_t)a, q = (int64_t)b;
  if (q == 0) return 0;
  if (q == -1) return 0ull - (uint64_t)p;
  int64_t r = p / q;
  if ((p % q != 0) && ((p < 0) != (q < 0))) r -= 1;
  return (uint64_t)r;
}

__device__ __forceinline__ uint64_t f_min(uint64_t a, uint64_t b, bool mn) {
  const double p = as_f64(a), q = as_f64(b);
  if (p != p) return a;
  if (q != q) return b;
  return f64_bits(mn ? (p <= q ? p : q) : (p >= q ? p : q));
}

__device__ __forceinline__ uint64_t i_min(uint64_t a, uint64_t b, bool mn) {
  const int64_t p = (int64_t)a, q = (int64_t)b;
  return (uint64_t)(mn ? (p < q ? p : q) : (p > q ? p : q));
}

__device__ __forceinline__ uint64_t i_abs(uint64_t a) {
  const int64_t p = (int64_t)a;
  return p < 0 ? (uint64_t)(0ull - (uint64_t)p) : (uint64_t)p;
}

}  // namespace lsbgen
