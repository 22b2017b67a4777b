// Peak microbenchmarks for the roofline denominators:
// fp64 DFMA throughput, HBM copy bandwidth, device properties.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
         x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
__global__ void dadd_loop(double* out, int iters, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
         x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 += b; x1 += b; x2 += b; x3 += b; x4 += b; x5 += b; x6 += b; x7 += b;
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int l2 = 0, clk = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"name\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"clock_khz\": %d, \"regs_per_sm\": %d, \"cc\": \"%d.%d\"}\n",
         p.name, p.multiProcessorCount, l2, p.sharedMemPerBlockOptin, clk, p.regsPerMultiprocessor, p.major, p.minor);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4000;
  for (int rep = 0; rep < 3; ++rep) {
    dfma_loop<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
    cudaEventRecord(e0);
    for (int k = 0; k < 10; ++k) dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 10.0 * blocks * threads * (double)iters * 16 * 8 * 2;
    printf("dfma rep%d: %.2f TFLOP/s (%.3f ms)\n", rep, fl / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    for (int k = 0; k < 10; ++k) dadd_loop<<<blocks, threads>>>(out, iters, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 10.0 * blocks * threads * (double)iters * 16 * 8;
    printf("dadd rep%d: %.2f Tinst/s\n", rep, ops / ms / 1e9);
  }
  size_t n = (size_t)1 << 27;  // 2 GiB per buffer
  double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    copy_k<<<p.multiProcessorCount * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy rep%d: %.1f GB/s\n", rep, 2.0 * n * 16 / ms / 1e6);
  }
  return 0;
}
