// pipe_overlap.cu -- do the fp64 pipe and the shared-memory (MIO) pipe of a
// B200 SM overlap?  (the FFT engine's time per element
// and pass is close to the SUM of its fp64 time and its exchange time.)
//
// One 256-thread CTA per SM (the row / pencil kernels' occupancy), a loop of
//   F: 16 independent DFMA chains per thread, K1 rounds
//   S: 16 STS.128 + 16 LDS.128 per thread (conflict-free, Stockham-exchange
//      volume: 32 bytes per element), K2 rounds
//   FS: both in one loop body on independent data
//   FSB: as FS with the exchange split by two CTA barriers (store, bar, load,
//        bar), as the engine's pass_exchange does
// and prints cycles per round.  If FS ~ max(F, S) the pipes overlap; if
// FS ~ F + S they do not.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_overlap tools/pipe_overlap.cu
#include <cuda_runtime.h>

#include <cstdio>

constexpr int E = 16, TH = 256;

template <bool FP, bool SH, bool BAR>
__global__ void __launch_bounds__(TH, 1) k(double* out, int rounds, double a, double b) {
  extern __shared__ double2 sm[];
  double x[E];
  double2 y[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    x[i] = threadIdx.x + i;
    y[i] = make_double2(i, threadIdx.x);
  }
  const int t = threadIdx.x;
  for (int r = 0; r < rounds; ++r) {
    if constexpr (FP) {
#pragma unroll
      for (int rep = 0; rep < 8; ++rep)
#pragma unroll
        for (int i = 0; i < E; ++i) x[i] = fma(x[i], a, b);
    }
    if constexpr (SH) {
#pragma unroll
      for (int i = 0; i < E; ++i) sm[t + TH * i] = y[i];
      if constexpr (BAR) __syncthreads();
#pragma unroll
      for (int i = 0; i < E; ++i) y[i] = sm[((t + 32) & (TH - 1)) + TH * ((i + 1) & (E - 1))];
      if constexpr (BAR) __syncthreads();
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < E; ++i) s += x[i] + y[i].x + y[i].y;
  if (s == 12345.678) out[0] = s;
}

template <bool FP, bool SH, bool BAR>
float run(const char* name, int rounds, double* out, int nsm) {
  const int smem = TH * E * 16;
  cudaFuncSetAttribute(k<FP, SH, BAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<FP, SH, BAR><<<nsm, TH, smem>>>(out, rounds, 1.0000001, 1e-9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<FP, SH, BAR><<<nsm, TH, smem>>>(out, rounds, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3 / rounds;
  // per round per SM: FP = 8 x 16 DFMA x 8 warps = 1024 warp-instructions
  // (512 cycles at 2 per cycle); SH = 2 x 16 x 4 wavefronts x 8 warps = 1024
  // wavefronts
  printf("%-4s %8.1f cycles per round (at the max clock)  [%s]\n", name, cyc, cudaGetErrorString(cudaGetLastError()));
  return (float)cyc;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int rounds = 20000;
  printf("per round per SM: F = 1024 DFMA warp-instructions, S = 512 STS.128 + 512 LDS.128 warp-instructions "
         "(2048 wavefronts)\n");
  const float f = run<true, false, false>("F", rounds, out, nsm);
  const float s = run<false, true, false>("S", rounds, out, nsm);
  const float sb = run<false, true, true>("SB", rounds, out, nsm);
  const float fs = run<true, true, false>("FS", rounds, out, nsm);
  const float fsb = run<true, true, true>("FSB", rounds, out, nsm);
  printf("FS  / (F + S)  = %.2f   FS  / max(F, S)  = %.2f\n", fs / (f + s), fs / (f > s ? f : s));
  printf("FSB / (F + SB) = %.2f   FSB / max(F, SB) = %.2f\n", fsb / (f + sb), fsb / (f > sb ? f : sb));
  return 0;
}
