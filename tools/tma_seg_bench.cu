// tma_seg_bench.cu -- read bandwidth of pencil-style TMA tile loads against
// the tile width W (columns of 16 bytes: the DRAM row segment is 16 W bytes).
// Each CTA walks down all rows of its W-column block in 64 KB sub-tiles
// through a ring of NST stages (TMA 2D boxes, mbarrier completion), as the
// K7/K8 pencil kernels do, with no arithmetic; neighbouring CTAs take
// neighbouring column blocks.  Prints GB/s per W.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_seg_bench tools/tma_seg_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstdlib>

constexpr int NST = 3;                 // stages of 64 KB
constexpr int STAGE = 64 * 1024;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128) k_load(const __grid_constant__ CUtensorMap map, int W, int rows, int ncb,
                                              int BR, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
  const int sub_rows = STAGE / (W * 16);                 // rows per sub-tile
  const int nsub = rows / sub_rows;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // this CTA's sequence of (column block, sub-tile) pairs
  const long per = (long)nsub;
  const long ncbs = (ncb - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const long total = ncbs * per;
  auto issue = [&](long j, int s) {
    const long cb = blockIdx.x + (j / per) * gridDim.x;
    const int r0 = (int)(j % per) * sub_rows;
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bars[s])),
                 "r"(STAGE)
                 : "memory");
    for (int b = 0; b < sub_rows; b += BR)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su(smem + s * STAGE + b * W * 16)),
          "l"(&map), "r"((int)(2 * W * cb)), "r"(r0 + b), "r"(su(&bars[s]))
          : "memory");
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < NST && s < total; ++s) issue(s, s);
  unsigned long long acc = 0;
  uint32_t ph[NST] = {};
  for (long j = 0; j < total; ++j) {
    const int s = (int)(j % NST);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su(&bars[s])),
        "r"(ph[s])
        : "memory");
    ph[s] ^= 1;
    acc += reinterpret_cast<const unsigned long long*>(smem + s * STAGE)[threadIdx.x];   // touch the stage
    __syncthreads();
    if (threadIdx.x == 0 && j + NST < total) issue(j + NST, s);
  }
  if (acc == 0x123456789ULL) *sink = acc;
}

// per-thread cp.async (16 bytes, L1 bypass) of the same sub-tiles: each thread
// copies elements threadIdx.x + 128 j of the [row][column] stage
__global__ void __launch_bounds__(128) k_cpasync(const double2* __restrict__ src, long cols, int W, int rows, int ncb,
                                                 unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int sub_rows = STAGE / (W * 16);
  const int nsub = rows / sub_rows;
  const long per = nsub;
  const long ncbs = (ncb - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const long total = ncbs * per;
  auto issue = [&](long j, int s) {
    const long cb = blockIdx.x + (j / per) * gridDim.x;
    const int r0 = (int)(j % per) * sub_rows;
    const int n = sub_rows * W;
    for (int e = threadIdx.x; e < n; e += 128) {
      const int r = e / W, c = e - r * W;
      const double2* g = src + (long)(r0 + r) * cols + cb * W + c;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(smem + s * STAGE + e * 16)), "l"(g) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < NST - 1 && s < total; ++s) issue(s, s);
  unsigned long long acc = 0;
  for (long j = 0; j < total; ++j) {
    const int s = (int)(j % NST);
    if (j + NST - 1 < total) issue(j + NST - 1, (int)((j + NST - 1) % NST));
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
    __syncthreads();
    acc += reinterpret_cast<const unsigned long long*>(smem + s * STAGE)[threadIdx.x];
    __syncthreads();
  }
  if (acc == 0x123456789ULL) *sink = acc;
}

// TMA tensor stores of the stage (bulk groups), W-column sub-tiles as in K7
__global__ void __launch_bounds__(128) k_store(const __grid_constant__ CUtensorMap map, int W, int rows, int ncb,
                                               int BR) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int sub_rows = STAGE / (W * 16);
  const int nsub = rows / sub_rows;
  const long per = nsub;
  const long ncbs = (ncb - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const long total = ncbs * per;
  for (long j = 0; j < total; ++j) {
    const int s = (int)(j % NST);
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NST - 1) : "memory");
      const long cb = blockIdx.x + (j / per) * gridDim.x;
      const int r0 = (int)(j % per) * sub_rows;
      for (int b = 0; b < sub_rows; b += BR)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&map),
                     "r"((int)(2 * W * cb)), "r"(r0 + b), "r"(su(smem + s * STAGE + b * W * 16))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  // rows x columns (default 2048 x 2^18: 4 MB row pitch) and extra pitch columns
  const int rows = argc > 2 ? atoi(argv[2]) : 2048;
  const long ucols = argc > 3 ? atol(argv[3]) : (1L << 18);
  const long cols = ucols + (argc > 1 ? atol(argv[1]) : 0);
  void* buf;
  if (cudaMalloc(&buf, (size_t)rows * cols * 16) != cudaSuccess) return 1;
  cudaMemset(buf, 1, (size_t)rows * cols * 16);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(fn);
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int smem = NST * STAGE + 64;
  cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("%d rows, row pitch %ld columns (%ld bytes)\n", rows, cols, cols * 16);
  std::vector<int> widths = {4, 8, 16};
  if (argc > 4) {                         // comma-separated widths, e.g. "1,2,4"
    widths.clear();
    for (const char* p = argv[4]; *p;) {
      widths.push_back(atoi(p));
      while (*p && *p != ',') ++p;
      if (*p == ',') ++p;
    }
  }
  for (int W : widths) {
    CUtensorMap map;
    const int BR = STAGE / (W * 16) < 256 ? STAGE / (W * 16) : 256;
    cuuint64_t dims[2] = {(cuuint64_t)(2 * cols), (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 16};
    cuuint32_t box[2] = {(cuuint32_t)(2 * W), (cuuint32_t)BR};
    cuuint32_t es[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("W=%d: encode failed\n", W);
      continue;
    }
    const int ncb = (int)(ucols / W);
    // TSB_SMS=<n>: use n CTAs (one per SM) instead of all SMs -- tells a
    // per-SM request-rate limit (GB/s scales with n) from a device-wide one
    const int nuse = getenv("TSB_SMS") ? atoi(getenv("TSB_SMS")) : nsm;
    for (int per_sm : {1}) {
      const int grid = nuse * per_sm;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      k_load<<<grid, 128, smem>>>(map, W, rows, ncb, BR, sink);
      cudaEventRecord(e0);
      const int reps = 3;
      for (int r = 0; r < reps; ++r) k_load<<<grid, 128, smem>>>(map, W, rows, ncb, BR, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gbs = (double)rows * ucols * 16 * reps / (ms / 1e3) / 1e9;
      printf("W=%2d (%3d-byte row segments, boxes %d x %d rows): TMA load %.1f GB/s  [%s]\n", W, 16 * W, W, BR, gbs,
             cudaGetErrorString(cudaGetLastError()));
      cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_cpasync<<<grid, 128, smem>>>((const double2*)buf, cols, W, rows, ncb, sink);
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) k_cpasync<<<grid, 128, smem>>>((const double2*)buf, cols, W, rows, ncb, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("        cp.async 16 B per thread: %.1f GB/s  [%s]\n",
             (double)rows * ucols * 16 * reps / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      cudaFuncSetAttribute(k_store, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_store<<<grid, 128, smem>>>(map, W, rows, ncb, BR);
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) k_store<<<grid, 128, smem>>>(map, W, rows, ncb, BR);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("        TMA store: %.1f GB/s  [%s]\n", (double)rows * ucols * 16 * reps / (ms / 1e3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
