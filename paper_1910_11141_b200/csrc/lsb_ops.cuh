// lsb_ops.cuh — per-lane device primitives of the B200 VM.
//
// Each function reproduces the arithmetic of the reference numpy kernel it
// replaces (reference pkg/src/lockstep/runtime.py and workloads.py), in the
// same evaluation order wherever numpy's order is deterministic:
//
//   rng_uniform        runtime.py:280-303     exact (64-bit integer hash)
//   dot                runtime.py:248-250     numpy pairwise add-reduce order
//   axpy               runtime.py:253-255     separate IEEE mul then add, never FMA
//   gaussian logpdf    workloads.py:188-189   np.einsum chunked sequential order
//   gaussian grad      workloads.py:191-192   -(x @ P); OpenBLAS order is not reproducible,
//                                             parity is 1e-12 relative
//   f64 -> i64         ndarray.astype(int64)  x86 cvttsd2si semantics (NaN/overflow -> INT64_MIN)
//
// Lane storage is "lane-minor": element i of one lane's vector lives at
// base[i * stride], so a warp touching element i of 32 lanes issues one
// coalesced 256-byte access.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lsb {

__device__ __forceinline__ double as_f64(uint64_t w) { return __longlong_as_double((long long)w); }

// asynchronous 8-byte global -> shared copy (LDGSTS): no register is held while in flight
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ uint64_t f64_bits(double x) { return (uint64_t)__double_as_longlong(x); }

// numpy float64 -> int64 cast on x86-64: truncation, and the "integer
// indefinite" value INT64_MIN for NaN and out-of-range inputs.
__device__ __forceinline__ int64_t f64_to_i64(double x) {
  if (!(x > -9223372036854775808.0 && x < 9223372036854775808.0)) {
    // x == -2^63 is representable and converts exactly
    return (x == -9223372036854775808.0) ? INT64_MIN : INT64_MIN;
  }
  return (int64_t)x;  // cvt.rzi.s64.f64 (truncation)
}

// runtime.rng_uniform: splitmix64 finaliser over key*A + counter*B (mod 2^64).
__device__ __forceinline__ double rng_uniform(int64_t key, int64_t ctr) {
  uint64_t z = (uint64_t)key * 0xA24BAED4963EE407ull + (uint64_t)ctr * 0x9E3779B97F4A7C15ull;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return __dmul_rn((double)(z >> 11), 1.0 / 9007199254740992.0);
}

// numpy pairwise_sum leaf (unroll 8, block 128) over p(i), i in [lo, lo+n), n <= 128.
template <class P>
__device__ __forceinline__ double pairwise_leaf(const P& p, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, p(lo + i));
    return r;
  }
  double r0 = p(lo + 0), r1 = p(lo + 1), r2 = p(lo + 2), r3 = p(lo + 3);
  double r4 = p(lo + 4), r5 = p(lo + 5), r6 = p(lo + 6), r7 = p(lo + 7);
  int i = 8;
  const int stop = n - (n % 8);
  for (; i < stop; i += 8) {
    r0 = __dadd_rn(r0, p(lo + i + 0)); r1 = __dadd_rn(r1, p(lo + i + 1));
    r2 = __dadd_rn(r2, p(lo + i + 2)); r3 = __dadd_rn(r3, p(lo + i + 3));
    r4 = __dadd_rn(r4, p(lo + i + 4)); r5 = __dadd_rn(r5, p(lo + i + 5));
    r6 = __dadd_rn(r6, p(lo + i + 6)); r7 = __dadd_rn(r7, p(lo + i + 7));
  }
  double r = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                       __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) r = __dadd_rn(r, p(lo + i));
  return r;
}

// numpy pairwise_sum over p(i), i in [lo, lo+n): blocks of <= 128 summed by
// pairwise_leaf, split at n2 = n/2 rounded down to a multiple of 8, left + right.
// The split tree is walked with an explicit stack (device recursion would put
// frames on the per-thread call stack, which overflows inside the VM kernels once
// n > 256); every addition happens in the recursive form's order. Out of line:
// one small frame, and the VM kernels do not inline a copy per call site.
template <class P>
__device__ __noinline__ double pairwise_split(const P& p, int lo, int n) {
  constexpr int kDepth = 32;  // n - n2 <= n/2 + 8: depth < 31 for any int n
  int s_lo[kDepth], s_n[kDepth];
  double s_left[kDepth];
  bool s_right[kDepth];
  int sp = 0;
  s_lo[0] = lo, s_n[0] = n, s_right[0] = false;
  for (;;) {
    // descend through left children to a leaf
    while (s_n[sp] > 128) {
      int n2 = s_n[sp] / 2;
      n2 -= n2 % 8;
      s_lo[sp + 1] = s_lo[sp], s_n[sp + 1] = n2, s_right[sp + 1] = false;
      ++sp;
    }
    double r = pairwise_leaf(p, s_lo[sp], s_n[sp]);
    // climb: a finished left child starts its sibling; a finished right child combines
    for (;;) {
      if (sp == 0) return r;
      const bool was_right = s_right[sp];
      --sp;
      if (!was_right) {
        int n2 = s_n[sp] / 2;
        n2 -= n2 % 8;
        s_left[sp] = r;
        s_lo[sp + 1] = s_lo[sp] + n2, s_n[sp + 1] = s_n[sp] - n2, s_right[sp + 1] = true;
        ++sp;
        break;
      }
      r = __dadd_rn(s_left[sp], r);
    }
  }
}

template <class P>
__device__ __forceinline__ double pairwise(const P& p, int lo, int n) {
  return n <= 128 ? pairwise_leaf(p, lo, n) : pairwise_split(p, lo, n);
}

struct StridedProd {
  const uint64_t* a;
  const uint64_t* b;
  int stride;
  __device__ double operator()(int i) const {
    return __dmul_rn(as_f64(a[(size_t)i * stride]), as_f64(b[(size_t)i * stride]));
  }
};

// (a*b).sum(axis=1): products rounded, then 0.0 + pairwise(products).
__device__ __forceinline__ double dot_lane(const uint64_t* a, const uint64_t* b, int n, int stride) {
  return __dadd_rn(0.0, pairwise(StridedProd{a, b, stride}, 0, n));
}

// logpdf of the equicorrelated gaussian, numpy einsum('zi,ij,zj->z') order:
// terms (x_i * P_ij) * x_j in i-major order, summed sequentially in chunks of
// (8192 // d) * d terms, each chunk from 0.0 into an accumulator from 0.0.
__device__ __forceinline__ double gauss_logpdf_exact(const uint64_t* x, int stride, int d,
                                                     const double* __restrict__ P, double norm) {
  const int chunk = (d <= 8192) ? (8192 / d) * d : d;
  double acc = 0.0, s = 0.0;
  int in_chunk = 0;
  for (int i = 0; i < d; ++i) {
    const double xi = as_f64(x[(size_t)i * stride]);
    const double* row = P + (size_t)i * d;
    for (int j = 0; j < d; ++j) {
      const double t = __dmul_rn(__dmul_rn(xi, __ldg(row + j)), as_f64(x[(size_t)j * stride]));
      s = __dadd_rn(s, t);
      if (++in_chunk == chunk) {
        acc = __dadd_rn(acc, s);
        s = 0.0;
        in_chunk = 0;
      }
    }
  }
  if (in_chunk) acc = __dadd_rn(acc, s);
  return __dsub_rn(norm, __dmul_rn(0.5, acc));
}

// numpy logaddexp(x, y) for float64 (npy_logaddexp): log1p/exp formulation.
__device__ __forceinline__ double np_logaddexp(double x, double y) {
  if (x == y) return x + 0.693147180559945309417232121458176568;  // NPY_LOGE2
  const double t = x - y;
  if (t > 0) return x + log1p(exp(-t));
  if (t <= 0) return y + log1p(exp(t));
  return t;  // NaN
}

// stable sigmoid(-m) exactly as workloads.logistic_regression.grad_fn writes it
__device__ __forceinline__ double lr_sig(double m) {
  if (m >= 0) {
    const double e = exp(-m);
    return e / (1.0 + e);
  }
  return 1.0 / (1.0 + exp(m));
}

// the same sigmoid(-m) without a divergent branch: exp(-|m|) is the exp both branches of
// lr_sig take, so every result is bit-identical
__device__ __forceinline__ double lr_sig_nb(double m) {
  const double e = exp(-fabs(m));
  return __ddiv_rn(m >= 0 ? e : 1.0, __dadd_rn(1.0, e));
}

}  // namespace lsb
