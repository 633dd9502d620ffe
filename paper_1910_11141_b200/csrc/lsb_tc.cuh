// lsb_tc.cuh — 5th-generation tensor core (tcgen05) helpers for sm_100a.
//
// Used by the fp32 arm's fused leapfrog (lsb_tc_leapfrog.cuh): the gradient
// contraction g = -(q P) as a 3xTF32 tcgen05.mma with
//   A = the warpgroup's 128 chains' positions, one chain per TMEM lane (K columns,
//       split q = hi + lo into two TF32 operands),
//   B = the target's precision matrix (hi/lo TF32 split) in shared memory, staged
//       once per CTA by a bulk (TMA) copy of a host-built image in the UMMA
//       K-major no-swizzle canonical layout,
//   D = fp32 accumulators in TMEM (128 lanes x N columns).
// Raw PTX only (no CUTLASS types); descriptor bit layouts follow the PTX ISA
// (tcgen05 instruction / shared-memory matrix descriptors).
#pragma once
#include <cstdint>
#include <cstring>
#include <vector>

namespace lsbtc {

// ---- host: TF32 rounding and the B operand image --------------------------------------------

// round-to-nearest-even to TF32 (10 explicit mantissa bits), as a float
inline float tf32_round_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) {  // finite
    const uint32_t lsb = (u >> 13) & 1u;
    u += 0x0fffu + lsb;
  }
  u &= 0xffffe000u;
  float y;
  std::memcpy(&y, &u, 4);
  return y;
}

// Byte offset of element (n, k) of a K-major operand in the no-swizzle canonical layout:
// 8-row x 16-byte core matrices; `lbo` bytes between core matrices adjacent in K,
// `sbo` bytes between 8-row groups (M/N).
inline int umma_nosw_offset(int n, int k, int lbo, int sbo) {
  return (n / 8) * sbo + (k / 4) * lbo + (n % 8) * 16 + (k % 4) * 4;
}

// Image of B[k][n] (fp32, row stride ldb, K x N) as two K-major TF32 operands, hi then lo
// (B = hi + lo): the MMA's B^T tile, N rows of K elements each. Returns bytes per operand.
inline int b_image_nosw(const float* B, int K, int N, int ldb, int lbo, int sbo, std::vector<uint8_t>& img) {
  const int bytes = ((N + 7) / 8) * sbo > ((K + 3) / 4) * lbo ? ((N + 7) / 8) * sbo : ((K + 3) / 4) * lbo;
  const int per = ((N + 7) / 8 - 1) * sbo + ((K + 3) / 4 - 1) * lbo + 128;
  const int size = per > bytes ? per : bytes;
  img.assign((size_t)2 * size, 0);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      const float x = B[(size_t)k * ldb + n];
      const float hi = tf32_round_host(x);
      const float lo = tf32_round_host(x - hi);
      const int off = umma_nosw_offset(n, k, lbo, sbo);
      std::memcpy(&img[off], &hi, 4);
      std::memcpy(&img[size + off], &lo, 4);
    }
  return size;
}

// ---- device ---------------------------------------------------------------------------------

#if defined(__CUDACC__)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float tf32_round(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

// whole-warp TMEM allocation (power of two >= 32 columns); the address lands in *dst
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
}

__device__ __forceinline__ void tmem_dealloc(uint32_t base, int cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols));
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra LAB_WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// the issuing thread's previously issued MMAs arrive on `bar` when complete
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// bulk global -> shared copy (TMA engine), completion counted in bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// warp-wide TMEM accesses: thread t touches lane (addr.lane + t), 8 consecutive columns
__device__ __forceinline__ void tmem_st8(uint32_t addr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(addr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(addr)
               : "memory");
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// instruction descriptor: kind::tf32, fp32 accumulate, A and B K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)                       // D format F32
         | (2u << 7)                     // A format TF32
         | (2u << 10)                    // B format TF32
         | ((uint32_t)(n >> 3) << 17)    // N / 8
         | ((uint32_t)(m >> 4) << 24);   // M / 16
}

// shared-memory matrix descriptor, K-major, no swizzle (layout type 0), sm_100 version 1
__device__ __forceinline__ uint64_t smem_desc_nosw(uint32_t addr, int lbo, int sbo) {
  return (uint64_t)((addr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}

// D[tmem] (+)= A[tmem] . B[smem]  (kind::tf32, one CTA)
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, int accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

#endif  // __CUDACC__

}  // namespace lsbtc
