// fp64_peaks.cu — microbenchmark of the B200 fp64 pipes the gradient can use:
// DFMA (SIMT) and DMMA (mma.sync.m8n8k4.f64 tensor path). MEASURED_PEAKS.json
// only carries bf16/HBM, so the fp64 roofline denominator is measured here.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// latency / issue-rate probe: `warps` warps of one CTA, each with ILP independent
// accumulator chains; reports SM cycles per DMMA per warp
template <int ILP>
__global__ void dmma_lat_kernel(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[ILP][2];
  for (int t = 0; t < ILP; ++t) { c[t][0] = 0; c[t][1] = 0; }
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < ILP; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < ILP; ++t) s += c[t][0] + c[t][1];
  const long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
void lat_probe(double* out, long long* dcyc) {
  for (int warps : {1, 4, 8, 16}) {
    const int iters = 4000;
    dmma_lat_kernel<ILP><<<1, 32 * warps>>>(out, dcyc, 10);
    dmma_lat_kernel<ILP><<<1, 32 * warps>>>(out, dcyc, iters);
    long long cyc = 0;
    cudaMemcpy(&cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
    printf("{\"probe\": \"dmma_latency\", \"ilp\": %d, \"warps_per_sm\": %d, \"cycles_per_dmma_per_warp\": %.2f}\n",
           ILP, warps, (double)cyc / ((double)iters * ILP));
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * 1 << 24);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    const int blocks = sms * (2048 / threads), iters = 2000;
    dfma_kernel<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("{\"pipe\": \"dfma\", \"threads\": %d, \"tflops\": %.2f}\n", threads, flops / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) {
    const int blocks = sms * (2048 / threads), iters = 2000;
    dmma_kernel<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf("{\"pipe\": \"dmma_m8n8k4\", \"threads\": %d, \"tflops\": %.2f}\n", threads, flops / ms / 1e9);
  }
  long long* dcyc;
  cudaMalloc(&dcyc, sizeof(long long));
  lat_probe<1>(out, dcyc);
  lat_probe<2>(out, dcyc);
  lat_probe<4>(out, dcyc);
  lat_probe<8>(out, dcyc);
  cudaError_t e = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
