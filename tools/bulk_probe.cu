// Bulk-copy ring microbenchmark (dev tool): one warp per CTA streams a buffer through a
// shared-memory ring of STAGES chunks with cp.async.bulk + mbarrier (the warp_lr_stream
// pattern), with no compute; prints the time per chunk for several chunk sizes / CTA counts.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o bulk_probe tools/bulk_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_1910_11141_b200/csrc/lsb_tc.cuh"

template <int STAGES, int MODE>
__global__ void ring(const double* src, size_t n_doubles, int chunk_doubles, double* out) {
  extern __shared__ __align__(128) double sm[];
  const int lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)STAGES * chunk_doubles);
  const int nch = (int)(n_doubles / chunk_doubles);
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) lsbtc::mbar_init(&bars[s], 1);
    lsbtc::fence_barrier_init();
  }
  __syncwarp();
  const uint32_t bytes = chunk_doubles * 8;
  auto issue = [&](int it) {
    const int st = it % STAGES;
    lsbtc::mbar_expect_tx(&bars[st], bytes);
    lsbtc::bulk_g2s(sm + (size_t)st * chunk_doubles, src + (size_t)(it % nch) * chunk_doubles, bytes, &bars[st]);
  };
  if (lane == 0)
    for (int it = 0; it < STAGES && it < nch; ++it) issue(it);
  double acc = 0.0;
  for (int it = 0; it < nch; ++it) {
    const int st = it % STAGES;
    const uint32_t par = (it / STAGES) & 1;
    if (MODE == 0) {
      lsbtc::mbar_wait(&bars[st], par);
    } else {  // test_wait spin
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(lsbtc::smem_u32(&bars[st])), "r"(par) : "memory");
    }
    acc += sm[(size_t)st * chunk_doubles + lane];
    __syncwarp();
    if (lane == 0 && it + STAGES < nch) issue(it + STAGES);
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  const size_t n = (size_t)100000 * 100;  // the config-4 design: 80 MB
  std::vector<double> h(n, 1.0);
  double *d, *o;
  cudaMalloc(&d, n * 8);
  cudaMalloc(&o, 8);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode)
    for (int cd : {112, 1600, 3200, 6400}) {
      for (int ctas : {1, 8, 148}) {
        const int smem = 4 * cd * 8 + 64;
        auto k = mode == 0 ? ring<4, 0> : ring<4, 1>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const size_t use = std::min(n, (size_t)cd * 4000);
        k<<<ctas, 32, smem>>>(d, use, cd, o);
        cudaEventRecord(e0);
        k<<<ctas, 32, smem>>>(d, use, cd, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double per = ms * 1e3 / (use / cd);
        printf("mode %d chunk %5d B ctas %3d: %.3f us/chunk, %.1f GB/s per warp (%s)\n", mode, cd * 8, ctas, per,
               cd * 8 / per / 1e3, cudaGetErrorString(cudaGetLastError()));
      }
    }
  return 0;
}
