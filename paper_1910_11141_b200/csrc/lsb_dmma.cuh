// lsb_dmma.cuh — warp-cooperative fp64 tensor-core contractions (DMMA m8n8k4).
//
// The gradient of the target is the only dense contraction on the path
// (reference workloads.py:191-192, 221-228). tcgen05 has no f64 kind; the
// fp64 tensor path on sm_100a is mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), and
// tools/fp64_peaks.cu measured it at 37.0 TFLOP/s on this pool's B200
// (DFMA 36.9) — the roofline denominator used by bench.py.
//
// One warp multiplies up to 8 chains (one m-tile, rows = chains) by the
// target matrix. The B operand is pre-swizzled on the host into fragment
// order, Bf[(ks * NT + nt) * 32 + lane] = B[4ks + lane%4][8nt + lane/4]
// (zero padded), so every B fragment is one coalesced 256-byte load. When the
// fragments fit, the warp engine stages them once per CTA in shared memory
// (SB = true: every warp of the SM reads one copy at LDS latency); otherwise
// they are read through L1 with evict_last priority.
//
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64):
//   A 8x4 row-major : lane holds A[lane/4][lane%4]
//   B 4x8 col-major : lane holds B[lane%4][lane/4]
//   C/D 8x8         : lane holds C[lane/4][2*(lane%4) + {0,1}]
#pragma once
#include <cstdint>

#ifndef LSB_BPF
#define LSB_BPF 0  // 1 = double-buffer the B fragments in registers
#endif

namespace lsb {

// read-only load with high L1 retention priority (the target matrix fragments)
__device__ __forceinline__ double ldg_keep(const double* p) {
  double v;
  asm("ld.global.nc.L1::evict_last.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}

// B-fragment load: SB = the fragments were staged in shared memory by the CTA
template <bool SB>
__device__ __forceinline__ double ld_b(const double* p) {
  if constexpr (SB) {
    double v;
    asm("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
  } else {
    return ldg_keep(p);
  }
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// acc[j] (n-tile nt0 + j) = sum_k A[row][k] * B[k][n] over k < 4*KS.
// `a_at(k)` returns this lane's A element for column k (row = lane/4).
template <int NTC, bool SB = false, class ALoad>
__device__ __forceinline__ void mtile_gemm(double (&acc)[NTC][2], const double* __restrict__ Bf,
                                           int KS, int NT, int nt0, const ALoad& a_at) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < NTC; ++j) acc[j][0] = acc[j][1] = 0.0;
  const double* bp = Bf + (size_t)nt0 * 32 + lane;
  const size_t kstride = (size_t)NT * 32;
#if LSB_BPF
  // fetch B one k-step ahead so the loads overlap the previous step's DMMAs
  double b_cur[NTC], b_next[NTC];
#pragma unroll
  for (int j = 0; j < NTC; ++j) b_cur[j] = ld_b<SB>(bp + j * 32);
  double a_next = a_at(lane & 3);
  for (int ks = 0; ks < KS; ++ks) {
    const double a = a_next;
    bp += kstride;
    if (ks + 1 < KS) {
      a_next = a_at(4 * (ks + 1) + (lane & 3));
#pragma unroll
      for (int j = 0; j < NTC; ++j) b_next[j] = ld_b<SB>(bp + j * 32);
    }
#pragma unroll
    for (int j = 0; j < NTC; ++j) dmma(acc[j], a, b_cur[j]);
#pragma unroll
    for (int j = 0; j < NTC; ++j) b_cur[j] = b_next[j];
  }
#else
  double a_next = a_at(lane & 3);
  for (int ks = 0; ks < KS; ++ks) {
    const double a = a_next;
    if (ks + 1 < KS) a_next = a_at(4 * (ks + 1) + (lane & 3));
#pragma unroll
    for (int j = 0; j < NTC; ++j) dmma(acc[j], a, ld_b<SB>(bp + j * 32));
    bp += kstride;
  }
#endif
}

// mtile_gemm with the A and B fragments of step k+1 loaded (into distinct
// registers) while step k's DMMAs run: the LDS latency hides behind the MMAs.
// For operands in shared memory (A tile and, with SB, the staged B fragments).
template <int NTC, bool SB, class ALoad>
__device__ __forceinline__ void mtile_gemm_pf(double (&acc)[NTC][2], const double* __restrict__ Bf,
                                              int KS, int NT, int nt0, const ALoad& a_at) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < NTC; ++j) acc[j][0] = acc[j][1] = 0.0;
  const double* bp = Bf + (size_t)nt0 * 32 + lane;
  const int kstride = NT * 32;
  double a = a_at(lane & 3), b[NTC];
#pragma unroll
  for (int j = 0; j < NTC; ++j) b[j] = ld_b<SB>(bp + j * 32);
#pragma unroll 1
  for (int ks = 0; ks + 1 < KS; ++ks) {
    bp += kstride;
    const double an = a_at(4 * (ks + 1) + (lane & 3));
    double bn[NTC];
#pragma unroll
    for (int j = 0; j < NTC; ++j) bn[j] = ld_b<SB>(bp + j * 32);
#pragma unroll
    for (int j = 0; j < NTC; ++j) dmma(acc[j], a, b[j]);
    a = an;
#pragma unroll
    for (int j = 0; j < NTC; ++j) b[j] = bn[j];
  }
#pragma unroll
  for (int j = 0; j < NTC; ++j) dmma(acc[j], a, b[j]);
}

// n-tiles per accumulator pass: 8 tiles = 16 fp64 accumulators per lane (32 registers)
#define LSB_NT_CHUNK 8

// Dispatch a runtime n-tile count (1..LSB_NT_CHUNK) to a compile-time template.
#define LSB_NT_DISPATCH(NTV, ...)                 \
  switch (NTV) {                                   \
    case 1: { constexpr int NTC = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int NTC = 2; __VA_ARGS__; } break;   \
    case 3: { constexpr int NTC = 3; __VA_ARGS__; } break;   \
    case 4: { constexpr int NTC = 4; __VA_ARGS__; } break;   \
    case 5: { constexpr int NTC = 5; __VA_ARGS__; } break;   \
    case 6: { constexpr int NTC = 6; __VA_ARGS__; } break;   \
    case 7: { constexpr int NTC = 7; __VA_ARGS__; } break;   \
    default: { constexpr int NTC = 8; __VA_ARGS__; } break; \
  }

}  // namespace lsb
