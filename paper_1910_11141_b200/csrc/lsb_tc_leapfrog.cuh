// lsb_tc_leapfrog.cuh — the fp32 arm's fused leapfrog superblock on 5th-generation tensor
// cores (included by lsb_vm.cuh inside namespace lsbvm).
//
// Same function as warp_leapfrog_rp (reference workloads.py:461-472: L leapfrog steps of
// g = -(q P), p = (e/2) g + p, q = e p + q, each multiply and add rounded separately),
// computed in float32 for the chains of a warpgroup at once: the warps of a warpgroup step
// independently and meet here (wg_rendezvous: every warp of the warpgroup that has not
// finished arrives at its next superblock step), then run one 128-row contraction:
//
//   TMEM (512 columns, one warpgroup at a time per CTA):
//     [  0, 128)  D  = q . P (fp32 accumulators, N = d rounded up to 16)
//     [128, 256)  Ah = TF32(q)          one chain per lane (lane 32 w + t = warp w's
//     [256, 384)  Al = TF32(q - Ah)     thread t), K = d rounded up to 8 columns
//     [384, 512)  p  (fp32 momentum)
//   shared memory: P_hi and P_lo (TF32 split of the fp32 precision matrix) in the UMMA
//     K-major no-swizzle layout, staged once per CTA by a bulk (TMA) copy.
//
// One gradient = 3 * K/8 tcgen05.mma kind::tf32 (Ah.Ph + Ah.Pl + Al.Ph: the 3xTF32 split,
// ~1e-6 relative, inside the fp32 contract of 1e-5 per leapfrog step), issued by one
// thread and committed to an mbarrier; the warps then apply the kicks/drift from TMEM.
// L+1 contractions per leaf (the duplicate gradient of consecutive steps is shared, as
// in the fp64 superblock). Values enter as f64 rounded to fp32 and leave as the f64 of
// the fp32 results.
#pragma once

#include "lsb_tc.cuh"

struct TcShared {
  uint32_t tmem;            // TMEM base address (512 columns)
  int lock;                 // 1 while a warpgroup owns the tensor memory
  uint32_t phase;           // parity of the next completion of mma_bar
  int pad;
  uint64_t mma_bar;
  uint64_t img_bar;
  // superblock rendezvous of each warpgroup's warps (wg_rendezvous / wg_leave)
  struct {
    int lock, arrived, gone, gen, mask, present;
  } rv[8];  // up to 32 warps per CTA
};
__shared__ TcShared lsb_tcs;

constexpr uint32_t kTcColD = 0, kTcColHi = 128, kTcColLo = 256, kTcColP = 384;

// named barrier of the `nthreads` threads of warpgroup wgi that take part in a superblock
__device__ __forceinline__ void wg_bar(int wgi, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + wgi), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void rv_lock(int* l) {
  while (atomicCAS(l, 0, 1) != 0) __nanosleep(32);
  __threadfence_block();
}
__device__ __forceinline__ void rv_unlock(int* l) {
  __threadfence_block();
  atomicExch(l, 0);
}

// Called by lane 0 with the warpgroup's rendezvous lock held: if every warp still running
// has arrived, release them together (present = their mask) and start a new generation.
__device__ __forceinline__ void rv_try_release(int wgi) {
  auto& r = lsb_tcs.rv[wgi];
  if (r.arrived > 0 && r.arrived + r.gone == 4) {
    r.present = r.mask;
    r.arrived = 0;
    r.mask = 0;
    __threadfence_block();
    atomicAdd(&r.gen, 1);
  }
}

// Whole warp: wait until every unfinished warp of this warpgroup is at its superblock step;
// returns the mask (bit = warp index within the warpgroup) of the warps taking part.
__device__ inline unsigned wg_rendezvous() {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wq = wid & 3, wgi = wid >> 2;
  unsigned present = 0;
  if (lane == 0) {
    auto& r = lsb_tcs.rv[wgi];
    rv_lock(&r.lock);
    const int gen = *(volatile int*)&r.gen;
    r.arrived += 1;
    r.mask |= 1 << wq;
    rv_try_release(wgi);
    rv_unlock(&r.lock);
    while (*(volatile int*)&r.gen == gen) __nanosleep(64);
    __threadfence_block();
    present = (unsigned)*(volatile int*)&r.present;
  }
  return __shfl_sync(0xffffffffu, present, 0);
}

// Whole warp, once when it stops stepping: peers no longer wait for it.
__device__ inline void wg_leave() {
  const int wid = threadIdx.x >> 5, wgi = wid >> 2;
  if ((threadIdx.x & 31) == 0) {
    auto& r = lsb_tcs.rv[wgi];
    rv_lock(&r.lock);
    r.gone += 1;
    rv_try_release(wgi);
    rv_unlock(&r.lock);
  }
  __syncwarp();
}

// Kernel prologue, every thread of the CTA: TMEM, barriers, the B image (bulk copy).
__device__ inline void tc_cta_begin(const VMArgs& a, unsigned char* dyn) {
  if (threadIdx.x == 0) {
    lsb_tcs.lock = 0;
    lsb_tcs.phase = 0;
    lsbtc::mbar_init(&lsb_tcs.mma_bar, 1);
    lsbtc::mbar_init(&lsb_tcs.img_bar, 1);
    lsbtc::fence_barrier_init();
  }
  if (threadIdx.x < 32) lsbtc::tmem_alloc(&lsb_tcs.tmem, 512);
  if (threadIdx.x < 8) {  // warps a short last warpgroup lacks never arrive: count them as gone
    const int nw = (int)(blockDim.x >> 5) - 4 * (int)threadIdx.x;
    lsb_tcs.rv[threadIdx.x] = {0, 0, nw >= 4 ? 0 : (nw > 0 ? 4 - nw : 4), 0, 0, 0};
  }
  lsbtc::tc_fence_before();
  __syncthreads();
  lsbtc::tc_fence_after();
  if (threadIdx.x == 0) {
    lsbtc::mbar_expect_tx(&lsb_tcs.img_bar, (uint32_t)a.tc_img_bytes);
    lsbtc::bulk_g2s(dyn + a.tc_smem_off, a.tc_img, (uint32_t)a.tc_img_bytes, &lsb_tcs.img_bar);
  }
  lsbtc::mbar_wait(&lsb_tcs.img_bar, 0);
}

// Kernel epilogue, every thread of the CTA.
__device__ inline void tc_cta_end() {
  lsbtc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    lsbtc::tc_fence_after();
    lsbtc::tmem_dealloc(lsb_tcs.tmem, 512);
  }
}

// q (f64 -> fp32) split into TF32 hi + lo
__device__ __forceinline__ void tc_split(float q, uint32_t& hi, uint32_t& lo) {
  const float h = lsbtc::tf32_round(q);
  hi = __float_as_uint(h);
  lo = __float_as_uint(__fsub_rn(q, h));
}

template <int KT>
__device__ void wg_leapfrog_tf32(const VMArgs& a, const Lane& ln, const ROp& op, bool part, long long chain) {
  extern __shared__ __align__(16) unsigned char lsb_dyn_u8[];
  constexpr int KP = 8 * KT;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wq = wid & 3, wgi = wid >> 2;
  const DevTarget& tg = a.targets[op.imm0];
  const int d = tg.dim, steps = op.imm1;
  const int NP = (d + 15) / 16 * 16;
  const int grow = (int)(op.bits & 0xffffffff), irow = (int)(op.bits >> 32);
  uint64_t* myq = part ? const_cast<uint64_t*>(ln.in(op, 0)) : nullptr;
  uint64_t* myp = part ? const_cast<uint64_t*>(ln.in(op, 1)) : nullptr;
  const bool wb = (op.kind & 1) != 0;
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
  // meet the warpgroup's other unfinished warps; the lowest present warp issues the MMAs
  const unsigned present = wg_rendezvous();
  const int nthr = 32 * __popc(present);
  const int issuer = __ffs(present) - 1;
  // own the CTA's tensor memory for this call
  if (wq == issuer && lane == 0)
    while (atomicCAS(&lsb_tcs.lock, 0, 1) != 0) __nanosleep(64);
  wg_bar(wgi, nthr);
  uint32_t phase = *(volatile uint32_t*)&lsb_tcs.phase;
  const uint32_t tbase = lsb_tcs.tmem;
  const uint32_t tb = tbase + ((uint32_t)(32 * wq) << 16);  // this warp's lane quarter
  const float e = __double2float_rn(mye);
  const float half = __fdiv_rn(e, 2.0f);
#pragma unroll 1
  for (int kt = 0; kt < KT; ++kt) {
    uint32_t hi[8], lo[8], pv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = 8 * kt + j;
      const bool in = part && k < d;
      tc_split(in ? __double2float_rn(as_f64(myq[(size_t)k * 32])) : 0.f, hi[j], lo[j]);
      pv[j] = __float_as_uint(in ? __double2float_rn(as_f64(myp[(size_t)k * 32])) : 0.f);
    }
    lsbtc::tmem_st8(tb + kTcColHi + 8 * kt, hi);
    lsbtc::tmem_st8(tb + kTcColLo + 8 * kt, lo);
    lsbtc::tmem_st8(tb + kTcColP + 8 * kt, pv);
  }
  lsbtc::tmem_st_wait();
  lsbtc::tc_fence_before();
  wg_bar(wgi, nthr);
  lsbtc::tc_fence_after();
  const uint32_t idesc = lsbtc::idesc_tf32(128, NP);
  const uint32_t bimg = lsbtc::smem_u32(lsb_dyn_u8 + a.tc_smem_off);
  double quad = 0.0;
  for (int pass = 0; steps > 0 && pass <= steps; ++pass) {
    if (pass > 0) {  // drift q = e p + q, split again for the next contraction
#pragma unroll 1
      for (int kt = 0; kt < KT; ++kt) {
        uint32_t hi[8], lo[8], pv[8];
        lsbtc::tmem_ld8(tb + kTcColHi + 8 * kt, hi);
        lsbtc::tmem_ld8(tb + kTcColLo + 8 * kt, lo);
        lsbtc::tmem_ld8(tb + kTcColP + 8 * kt, pv);
        lsbtc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float q = __fadd_rn(__uint_as_float(hi[j]), __uint_as_float(lo[j]));
          tc_split(__fadd_rn(__fmul_rn(e, __uint_as_float(pv[j])), q), hi[j], lo[j]);
        }
        lsbtc::tmem_st8(tb + kTcColHi + 8 * kt, hi);
        lsbtc::tmem_st8(tb + kTcColLo + 8 * kt, lo);
      }
      lsbtc::tmem_st_wait();
      lsbtc::tc_fence_before();
      wg_bar(wgi, nthr);
      lsbtc::tc_fence_after();
    }
    if (wq == issuer && lane == 0) {  // D = q . P on the tensor cores (3xTF32)
#pragma unroll 1
      for (int ks = 0; ks < KT; ++ks) {
        const uint64_t bh = lsbtc::smem_desc_nosw(bimg + ks * 2 * a.tc_lbo, a.tc_lbo, a.tc_sbo);
        const uint64_t bl = lsbtc::smem_desc_nosw(bimg + a.tc_half_bytes + ks * 2 * a.tc_lbo, a.tc_lbo, a.tc_sbo);
        lsbtc::mma_tf32_ts(tbase + kTcColD, tbase + kTcColHi + 8 * ks, bh, idesc, ks > 0);
        lsbtc::mma_tf32_ts(tbase + kTcColD, tbase + kTcColHi + 8 * ks, bl, idesc, 1);
        lsbtc::mma_tf32_ts(tbase + kTcColD, tbase + kTcColLo + 8 * ks, bh, idesc, 1);
      }
      lsbtc::mma_commit(&lsb_tcs.mma_bar);
    }
    __syncwarp();
    lsbtc::mbar_wait(&lsb_tcs.mma_bar, phase);
    phase ^= 1u;
    lsbtc::tc_fence_after();
    const bool last = pass == steps;
    const int nkick = (pass == 0 || last) ? 1 : 2;
#pragma unroll 1
    for (int kt = 0; kt < KT; ++kt) {
      uint32_t dv[8], pv[8], hi[8], lo[8];
      lsbtc::tmem_ld8(tb + kTcColD + 8 * kt, dv);
      lsbtc::tmem_ld8(tb + kTcColP + 8 * kt, pv);
      if (last) {
        lsbtc::tmem_ld8(tb + kTcColHi + 8 * kt, hi);
        lsbtc::tmem_ld8(tb + kTcColLo + 8 * kt, lo);
      }
      lsbtc::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float g = -__uint_as_float(dv[j]);
        float p = __fadd_rn(__fmul_rn(half, g), __uint_as_float(pv[j]));
        if (nkick == 2) p = __fadd_rn(__fmul_rn(half, g), p);
        pv[j] = __float_as_uint(p);
        const int k = 8 * kt + j;
        if (last && part && k < d) {
          if (my_g != nullptr) my_g[(size_t)k * 32] = f64_bits((double)g);
          const float q = __fadd_rn(__uint_as_float(hi[j]), __uint_as_float(lo[j]));
          quad = fma((double)q, (double)__uint_as_float(dv[j]), quad);
        }
      }
      lsbtc::tmem_st8(tb + kTcColP + 8 * kt, pv);
    }
    lsbtc::tmem_st_wait();
    lsbtc::tc_fence_before();
    wg_bar(wgi, nthr);  // D is consumed before the next contraction overwrites it
    lsbtc::tc_fence_after();
  }
  // write back q, p and _ret = vcat(q, p) (each thread its own chain: coalesced rows)
#pragma unroll 1
  for (int kt = 0; kt < KT; ++kt) {
    uint32_t hi[8], lo[8], pv[8];
    lsbtc::tmem_ld8(tb + kTcColHi + 8 * kt, hi);
    lsbtc::tmem_ld8(tb + kTcColLo + 8 * kt, lo);
    lsbtc::tmem_ld8(tb + kTcColP + 8 * kt, pv);
    lsbtc::tmem_ld_wait();
    if (part) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = 8 * kt + j;
        if (k < d) {
          const uint64_t qv = f64_bits((double)__fadd_rn(__uint_as_float(hi[j]), __uint_as_float(lo[j])));
          const uint64_t pw = f64_bits((double)__uint_as_float(pv[j]));
          if (wb) {
            myq[(size_t)k * 32] = qv;
            myp[(size_t)k * 32] = pw;
          }
          my_ret[(size_t)k * 32] = qv;
          my_ret[(size_t)(d + k) * 32] = pw;
        }
      }
    }
  }
  if (part && want_lp) my_lp[0] = f64_bits(gauss_lp_from_quad(tg.norm, quad));
  lsbtc::tc_fence_before();
  wg_bar(wgi, nthr);
  if (wq == issuer && lane == 0) {
    lsb_tcs.phase = phase;
    __threadfence_block();
    atomicExch(&lsb_tcs.lock, 0);
  }
  (void)KP;
}

// fp32 arm dispatch for d <= 128 (KT = ceil(d / 8) k-tiles of 8)
__device__ inline void wg_leapfrog_tf32_any(const VMArgs& a, const Lane& ln, const ROp& op, bool part,
                                            long long chain) {
  switch ((a.targets[op.imm0].dim + 7) / 8) {
#define LSB_TC_CASE(K) \
  case K: wg_leapfrog_tf32<K>(a, ln, op, part, chain); return;
    LSB_TC_CASE(1) LSB_TC_CASE(2) LSB_TC_CASE(3) LSB_TC_CASE(4) LSB_TC_CASE(5) LSB_TC_CASE(6)
    LSB_TC_CASE(7) LSB_TC_CASE(8) LSB_TC_CASE(9) LSB_TC_CASE(10) LSB_TC_CASE(11) LSB_TC_CASE(12)
    LSB_TC_CASE(13) LSB_TC_CASE(14) LSB_TC_CASE(15) LSB_TC_CASE(16)
#undef LSB_TC_CASE
    default: break;
  }
}
