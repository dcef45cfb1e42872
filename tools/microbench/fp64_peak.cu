// FP64 peaks of this B200: DMMA (mma.sync.m16n8k4.f64, the FP64 tensor path;
// tcgen05 has no f64 kind) and DFMA (CUDA cores).  Each warp runs 8
// independent accumulator chains in registers, no memory traffic; grid =
// 148 SMs x `blocks_per_sm` CTAs of 256 threads.  Prints TFLOP/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dmma_kernel(double* out, int iters) {
  double d[8][4];
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, b0 = 1.0 - a0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) d[i][e] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(d[i][0]), "+d"(d[i][1]), "+d"(d[i][2]), "+d"(d[i][3])
                   : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) s += d[i][e];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters) {
  double d[8];
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = fma(d[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 4096);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bps : {1, 2, 4}) {
    const int grid = nsm * bps, iters = 20000;
    dmma_kernel<<<grid, 256>>>(out, 100);
    cudaEventRecord(e0);
    dmma_kernel<<<grid, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 16 * 8 * 4 * 8.0 * iters * (grid * 8.0);
    printf("{\"kernel\": \"dmma_m16n8k4\", \"ctas_per_sm\": %d, \"tflops\": %.2f}\n", bps, fl / (ms * 1e-3) / 1e12);
    dfma_kernel<<<grid, 256>>>(out, 100);
    cudaEventRecord(e0);
    dfma_kernel<<<grid, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl2 = 2.0 * 32 * iters * (grid * 256.0);
    printf("{\"kernel\": \"dfma\", \"ctas_per_sm\": %d, \"tflops\": %.2f}\n", bps, fl2 / (ms * 1e-3) / 1e12);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
