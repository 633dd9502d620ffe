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

// dst[i] = f(i) for i < W, 8 loads in flight before the stores
template <int W, class F>
__device__ __forceinline__ void ew(uint64_t* dst, const F& f) {
  constexpr int full = W / 8 * 8;
#pragma unroll 1
  for (int i = 0; i < full; i += 8) {
    uint64_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = f(i + j);
#pragma unroll
    for (int j = 0; j < 8; ++j) dst[(i + j) * S] = v[j];
  }
#pragma unroll
  for (int i = full; i < W; ++i) dst[i * S] = f(i);
}

template <int W>
__device__ __forceinline__ void copy(uint64_t* dst, const uint64_t* src) {
  if (dst != src) ew<W>(dst, [&](int i) { return src[i * S]; });
}

template <int W>
__device__ __forceinline__ void fill(uint64_t* dst, uint64_t v) {
  ew<W>(dst, [&](int) { return v; });
}

template <int W>
__device__ __forceinline__ void axpy(uint64_t* dst, double s, const uint64_t* x, const uint64_t* y) {
  ew<W>(dst, [&](int i) { return f64_bits(__dadd_rn(__dmul_rn(s, as_f64(x[i * S])), as_f64(y[i * S]))); });
}

template <int W>
__device__ __forceinline__ void select(uint64_t* dst, bool c, const uint64_t* x, const uint64_t* y) {
  const uint64_t* src = c ? x : y;
  if (src != dst) ew<W>(dst, [&](int i) { return src[i * S]; });
}

template <int W>
__device__ __forceinline__ double dot(const uint64_t* x, const uint64_t* y) {
  return lsb::dot_lane(x, y, W, S);
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
