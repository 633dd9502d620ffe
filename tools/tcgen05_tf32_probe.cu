// tcgen05 kind::tf32 probe (dev tool): D[128 x N] = A[128 x K] . B[K x N] with A in TMEM
// (one chain per lane, K columns), B in shared memory (K-major, no swizzle: 8-row x 16-byte
// core matrices), D in TMEM (fp32). Checks plain TF32 and the 3xTF32 split against fp64.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/tcgen05_tf32_probe tools/tcgen05_tf32_probe.cu
//   tools/bin/tcgen05_tf32_probe
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../paper_1910_11141_b200/csrc/lsb_tc.cuh"

using namespace lsbtc;

constexpr int M = 128;
constexpr int K = 104;  // padded to a multiple of 8
constexpr int N = 112;  // padded to a multiple of 16

__global__ void __launch_bounds__(128, 1) probe(const float* A, const uint8_t* Bimg, int bbytes, float* D,
                                                int lbo, int sbo, int split) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < bbytes / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = reinterpret_cast<const uint32_t*>(Bimg)[i];
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  if (threadIdx.x == 0) mbar_init(&mbar, 1);
  fence_barrier_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;
  const int row = 32 * warp + lane;
  const uint32_t lane_addr = (uint32_t)(32 * warp) << 16;
  // A hi / lo into columns [128, 128+K) and [256, 256+K)
  for (int k0 = 0; k0 < K; k0 += 8) {
    uint32_t hi[8], lo[8];
    for (int j = 0; j < 8; ++j) {
      const float x = A[row * K + k0 + j];
      const float h = tf32_round(x);
      hi[j] = __float_as_uint(h);
      lo[j] = __float_as_uint(tf32_round(x - h));
    }
    tmem_st8(tb + lane_addr + 128 + k0, hi);
    tmem_st8(tb + lane_addr + 256 + k0, lo);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    const uint32_t bsmem = smem_u32(smem);
    const int half = bbytes / 2;  // image: B_hi then B_lo
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint64_t bhi = smem_desc_nosw(bsmem + ks * 2 * lbo, lbo, sbo);
      const uint64_t blo = smem_desc_nosw(bsmem + half + ks * 2 * lbo, lbo, sbo);
      mma_tf32_ts(tb + 0, tb + 128 + 8 * ks, bhi, idesc, ks > 0);
      if (split) {
        mma_tf32_ts(tb + 0, tb + 128 + 8 * ks, blo, idesc, 1);
        mma_tf32_ts(tb + 0, tb + 256 + 8 * ks, bhi, idesc, 1);
      }
    }
    mma_commit(&mbar);
  }
  __syncwarp();
  mbar_wait(&mbar, 0);
  tc_fence_after();
  for (int n0 = 0; n0 < N; n0 += 8) {
    uint32_t v[8];
    tmem_ld8(tb + lane_addr + n0, v);
    tmem_ld_wait();
    for (int j = 0; j < 8; ++j) D[row * N + n0 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

int main() {
  std::vector<float> A(M * K, 0.f), B(K * N, 0.f);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xffff) / 32768.0f - 1.0f; };
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < 100; ++k) A[m * K + k] = rnd();
  for (int k = 0; k < 100; ++k)
    for (int n = 0; n < 100; ++n) B[k * N + n] = rnd() * 0.37f;
  std::vector<double> ref(M * N, 0.0);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0;
      for (int k = 0; k < K; ++k) acc += (double)A[m * K + k] * (double)B[k * N + n];
      ref[m * N + n] = acc;
    }
  float *dA, *dD;
  uint8_t* dB;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  const int variants[][2] = {{128, (K / 4) * 128}, {(N / 8) * 128, 128}};
  for (auto& v : variants) {
    const int lbo = v[0], sbo = v[1];
    std::vector<uint8_t> img;
    const int bytes = b_image_nosw(B.data(), K, N, N, lbo, sbo, img);  // hi then lo
    cudaMalloc(&dB, img.size());
    cudaMemcpy(dB, img.data(), img.size(), cudaMemcpyHostToDevice);
    for (int split = 0; split < 2; ++split) {
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)img.size());
      cudaMemset(dD, 0, M * N * 4);
      probe<<<1, 128, img.size()>>>(dA, dB, (int)img.size(), dD, lbo, sbo, split);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> D(M * N);
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, mx = 0;
      for (int i = 0; i < M * N; ++i) {
        err = std::max(err, std::fabs(D[i] - ref[i]));
        mx = std::max(mx, std::fabs(ref[i]));
      }
      printf("lbo %5d sbo %5d split %d: %s max abs err %.3e (rel to max %.3e)  D[0..3] %f %f %f / ref %f %f %f\n",
             lbo, sbo, split, cudaGetErrorString(e), err, err / mx, D[0], D[1], D[2], ref[0], ref[1], ref[2]);
      (void)bytes;
    }
    cudaFree(dB);
  }
  return 0;
}
