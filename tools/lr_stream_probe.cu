// warp_lr_stream in isolation, with parts switched off (V bits: 1 no sigmoid, 2 no G GEMM,
// 4 no margin GEMM) (dev tool): one warp per CTA, one gradient call over a tall design, timed
// with CUDA events — separates the kernel's own speed from the VM context. lrs_v is a
// snapshot of warp_lr_stream_body (csrc/lsb_vm.cuh) with those switches added; re-take it
// after changing the kernel.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include \
//        -o lr_stream_probe tools/lr_stream_probe.cu
#include <cstdio>
#include <vector>
#include "../paper_1910_11141_b200/csrc/lsb_vm.cuh"
using namespace lsbvm;
namespace lsbvm {
template <int NT2, bool LOGPDF, int V>
__device__ __noinline__ void lrs_v(const DevTarget& tgr, bool part, const uint64_t* xp, uint64_t* dst,
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
      for (int ks = 0; ks < ((V & 4) ? 0 : KS); ks += 2) {
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
      const double s0 = 8 * t + 2 * c < pts ? ((V & 1) ? m0 : lsb::lr_sig_nb(m0)) : 0.0;
      const double s1 = 8 * t + 2 * c + 1 < pts ? ((V & 1) ? m1 : lsb::lr_sig_nb(m1)) : 0.0;
      const double u0 = __shfl_sync(kFull, s0, q0), u1 = __shfl_sync(kFull, s1, q0);
      const double v0 = __shfl_sync(kFull, s0, q1), v1 = __shfl_sync(kFull, s1, q1);
      const double a0 = hi ? u1 : u0, a1 = hi ? v1 : v0;
      const bool r0 = 8 * t + c < pts, r1 = 8 * t + 4 + c < pts;
      const double* b0 = X + (size_t)(8 * t + c) * d + g;
      const double* b1 = b0 + (size_t)4 * d;
#pragma unroll
      for (int j = 0; j < ((V & 2) ? 0 : NT2); ++j) {
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

}  // namespace lsbvm

template <int NT2, int V>
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ DevTarget tg, const uint64_t* x, uint64_t* y) {
  extern __shared__ double sm[];
  const int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  const uint64_t* xp = x + (size_t)w * tg.dim * 32 + lane;
  uint64_t* dp = y + (size_t)w * tg.dim * 32 + lane;
  lrs_v<NT2, false, V>(tg, true, xp, dp, sm + (threadIdx.x / 32) * lr_stream_doubles(tg.dim));
}

template <int NT2, int V = 0>
void run(int n, int d, int warps) {
  std::vector<double> h((size_t)n * d);
  for (size_t i = 0; i < h.size(); ++i) h[i] = ((i * 2654435761u) % 1000) / 1000.0 - 0.5;
  DevTarget tg{};
  tg.kind = 2; tg.dim = d; tg.n = n; tg.NT2 = NT2;
  double* P;
  cudaMalloc(&P, h.size() * 8);
  cudaMemcpy(P, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  tg.P = P;
  uint64_t *x, *y;
  cudaMalloc(&x, (size_t)warps * d * 32 * 8);
  cudaMalloc(&y, (size_t)warps * d * 32 * 8);
  cudaMemset(x, 0, (size_t)warps * d * 32 * 8);
  const int smem = lr_stream_doubles(d) * 8;
  cudaFuncSetAttribute(k<NT2, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<NT2, V><<<warps, 32, smem>>>(tg, x, y);
  cudaEventRecord(e0);
  k<NT2, V><<<warps, 32, smem>>>(tg, x, y);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const int chunks = 4 * ((n + 15) / 16);  // per 16 points
  printf("V=%d n=%d d=%d NT2=%d warps=%d: %.3f ms, %.3f us/chunk, %.1f GB/s per warp (%s)\n", V, n, d, NT2, warps, ms,
         ms * 1e3 / chunks, 4.0 * n * d * 8 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<13, 0>(100000, 100, 1);
  run<13, 1>(100000, 100, 1);
  run<13, 2>(100000, 100, 1);
  run<13, 3>(100000, 100, 1);
  run<13, 7>(100000, 100, 1);
  run<1, 0>(20001, 7, 1);
  run<1, 1>(20001, 7, 1);
  run<1, 7>(20001, 7, 1);
  return 0;
}
