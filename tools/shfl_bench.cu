// Microbenchmark: warp-shuffle vs shared-memory exchange throughput per SM on
// B200 (decides whether the FFT engine's last exchange should be shuffles).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o shfl_bench shfl_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_shfl(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      a0 = __shfl_xor_sync(0xffffffffu, a0, m); a1 = __shfl_xor_sync(0xffffffffu, a1, m);
      a2 = __shfl_xor_sync(0xffffffffu, a2, m); a3 = __shfl_xor_sync(0xffffffffu, a3, m);
      a4 = __shfl_xor_sync(0xffffffffu, a4, m); a5 = __shfl_xor_sync(0xffffffffu, a5, m);
      a6 = __shfl_xor_sync(0xffffffffu, a6, m); a7 = __shfl_xor_sync(0xffffffffu, a7, m);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_smem(double* out, int iters) {
  __shared__ double2 buf[256 * 8 + 64];
  double2 v[8];
  for (int i = 0; i < 8; ++i) v[i] = make_double2(threadIdx.x + i, i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) buf[i * 256 + threadIdx.x] = v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = buf[((i + 1) & 7) * 256 + (threadIdx.x ^ 1)];
    __syncthreads();
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += v[i].x + v[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 1024 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int threads : {256, 512, 1024}) {
    const int iters = 2000;
    k_shfl<<<sms, threads>>>(out, 10);
    cudaEventRecord(a);
    k_shfl<<<sms, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    // 8 doubles x 5 masks = 80 32-bit shuffles per thread per iteration
    double shfl_warp = (double)iters * 80 * (threads / 32);
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("shfl  threads=%4d: %.3f warp-shfl(32b) per SM-cycle  (%.2f ms)\n", threads, shfl_warp / cyc, ms);
    if (threads > 256) continue;
    k_smem<<<sms, 256>>>(out, 10);
    cudaEventRecord(a);
    k_smem<<<sms, 256>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    // per iteration per warp: 8 STS.128 + 8 LDS.128 = 64 wavefronts at 128 B each
    double wf = (double)iters * 64 * 8;
    cyc = ms * 1e-3 * clk * 1e3;
    printf("smem  threads= 256: %.3f wavefronts(128B) per SM-cycle (%.2f ms)\n", wf / cyc, ms);
  }
  // two CTAs of 256 per SM for smem
  {
    const int iters = 2000;
    float ms;
    cudaEventRecord(a);
    k_smem<<<2 * sms, 256>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double wf = (double)iters * 64 * 16;
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("smem  2x256/SM:     %.3f wavefronts(128B) per SM-cycle (%.2f ms)\n", wf / cyc, ms);
  }
  return 0;
}
