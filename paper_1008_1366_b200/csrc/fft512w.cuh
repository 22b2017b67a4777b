// fft512w.cuh -- warp-resident 512-point fp64 FFT: one shared-memory
// transpose plus one warp-shuffle radix-2 stage (device functions, sm_100a).
//
// The Stockham engine of fft_dev.cuh needs two shared-memory exchanges per
// 512-point transform (passes 16 x 16 x 2, or 8 x 8 x 8); at m = 512 the row
// and pencil kernels of the 3D configs are bound by the SM's shared-memory
// wavefronts (ncu r02: K3<512> 80% of the L1/shared pipe), and one exchange
// (a 16-byte STS + LDS per element, 8 wavefronts per warp-element) is the
// largest part of that traffic.  Here a warp owns one 512-point vector, lane
// n2 (0..31) holding x[n2 + 32 n1], n1 = 0..15 (the natural strided
// distribution of fft_dev.cuh with E = 16), and N = 16 x 32 is split as
//
//   backward (SIGN = +1, "bwd"):
//     1. DFT16 over n1 in registers:        A[n2, k1]
//     2. twiddle w512^{n2 k1}
//     3. transpose through shared memory:   lane (k1, b) gets A[b + 2a, k1], a = 0..15
//     4. DFT16 over a in registers:         Y_b[k2'], k2' = 0..15
//     5. radix-2 over b across the lane pair (k1, 0) / (k1, 1) with warp
//        shuffles (8 of the 16 values cross, 4 x 32-bit shuffles each):
//        X[k1 + 16 k2] = Y_0[k2'] + (-1)^c w32^{k2'} Y_1[k2'],  k2 = k2' + 16 c
//   and the output stays in the lane-pair order sigma: lane L = 2 k1 + b,
//   element e = j + 8 c (j < 8, c < 2) holds X[k1 + 16 (8 b + j + 16 c)].
//
//   forward (SIGN = -1, "fwd"): the exact reverse (radix-2 across the pair,
//   DFT16, transpose back, twiddle, DFT16), consuming sigma and producing the
//   natural strided order.
//
// A pointwise product between a bwd and a fwd transform is order-independent
// ("the scrambled Fourier subtransforms ... can be multiplied
// together as they are produced"), so kernels chain bwd -> product -> fwd in
// registers.  Per transform: one exchange (128 wavefronts per warp) and 32
// shuffles instead of two exchanges (256 wavefronts); measured on B200
// (tools/shfl_bench.cu): one 32-bit warp shuffle per SM cycle, 0.9 128-byte
// shared wavefronts per SM cycle.
#pragma once
#include "fft_dev.cuh"

namespace idc {

namespace w512 {

constexpr int N = 512, E = 16, LANES = 32;
constexpr int ROW = 34;                      // padded transpose row (16-byte slots): conflict-free both ways
constexpr int XB = 16 * ROW;                 // exchange slots per warp

__device__ __forceinline__ double shfl_x1(double v) { return __shfl_xor_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double2 shfl_pair(double2 v) { return make_double2(shfl_x1(v.x), shfl_x1(v.y)); }
__device__ __forceinline__ double2 sel2(bool p, double2 a, double2 b) { return p ? a : b; }

// step 2 twiddles: x[k1] * w512^{SIGN n2 k1}, k1 = 1..15, from the table
// tw[(k1 - 1) * 32 + n2] = exp(+2 pi i n2 k1 / 512) (tables.cu warp512_table)
template <int SIGN>
__device__ __forceinline__ void twiddle(double2 (&v)[E], int n2, const double2* __restrict__ tw) {
#pragma unroll
  for (int k1 = 1; k1 < E; ++k1) v[k1] = cmul_dir<SIGN>(v[k1], ldtw_pass(&tw[(k1 - 1) * LANES + n2]));
}

}  // namespace w512

// Backward 512-point transform of the warp's vector (natural strided in,
// sigma out).  xw: this warp's XB exchange slots; lane = lane index 0..31;
// tw = warp512_table().  Contains two __syncwarp()s.
template <int SIGN = +1>
__device__ __forceinline__ void fft512w_bwd(double2 (&v)[16], int lane, double2* __restrict__ xw,
                                            const double2* __restrict__ tw) {
  using namespace w512;
  dft<16, SIGN>(v);                                         // 1. over n1
  twiddle<SIGN>(v, lane, tw);                               // 2.
#pragma unroll
  for (int k1 = 0; k1 < E; ++k1) xw[k1 * ROW + lane] = v[k1];   // 3. transpose
  __syncwarp();
  const int k1 = lane >> 1, b = lane & 1;
#pragma unroll
  for (int a = 0; a < E; ++a) v[a] = xw[k1 * ROW + b + 2 * a];
  __syncwarp();
  dft<16, SIGN>(v);                                         // 4. over a -> Y_b[k2']
  // 5. lane b = 0 keeps k2' = j, lane b = 1 keeps k2' = 8 + j (j < 8)
  static_for<8>([&](auto J) {
    constexpr int j = decltype(J)::value;
    const double2 send = sel2(b, v[j], v[8 + j]);          // b=1 sends Y_1[j], b=0 sends Y_0[8+j]
    const double2 recv = shfl_pair(send);
    const double2 y0 = sel2(b, recv, v[j]);                 // Y_0[8b + j]
    double2 y1 = twc<j, 32, SIGN>(sel2(b, v[8 + j], recv)); // w32^{j} Y_1[8b + j] ...
    if (b) y1 = mul_i<SIGN>(y1);                            // ... times w32^{8 b} = (SIGN i)^b
    v[j] = cadd(y0, y1);                                    // c = 0
    v[8 + j] = csub(y0, y1);                                // c = 1
  });
}

// Forward 512-point transform (sigma in, natural strided out).
template <int SIGN = -1>
__device__ __forceinline__ void fft512w_fwd(double2 (&v)[16], int lane, double2* __restrict__ xw,
                                            const double2* __restrict__ tw) {
  using namespace w512;
  const int k1 = lane >> 1, b = lane & 1;
  // 5'. Z_0[k2'] = X[k2'] + X[k2' + 16], Z_1[k2'] = w32^{SIGN k2'} (X[k2'] - X[k2' + 16]), k2' = 8b + j
  static_for<8>([&](auto J) {
    constexpr int j = decltype(J)::value;
    const double2 s = cadd(v[j], v[8 + j]);
    double2 d = twc<j, 32, SIGN>(csub(v[j], v[8 + j]));
    if (b) d = mul_i<SIGN>(d);
    const double2 recv = shfl_pair(sel2(b, s, d));          // b=0 sends Z_1[j], b=1 sends Z_0[8+j]
    v[j] = sel2(b, recv, s);                                // b=0: Z_0[j];     b=1: Z_1[j]
    v[8 + j] = sel2(b, d, recv);                            // b=0: Z_0[8+j];   b=1: Z_1[8+j]
  });
  dft<16, SIGN>(v);                                         // 4'. over k2' -> B[b + 2a, k1]
#pragma unroll
  for (int a = 0; a < E; ++a) xw[k1 * ROW + b + 2 * a] = v[a];   // 3'. transpose back
  __syncwarp();
#pragma unroll
  for (int kk = 0; kk < E; ++kk) v[kk] = xw[kk * ROW + lane];
  __syncwarp();
  twiddle<SIGN>(v, lane, tw);                               // 2'.
  dft<16, SIGN>(v);                                         // 1'. over k1 -> x[lane + 32 n1]
}

// sigma: the frequency index held by (lane, element e) after fft512w_bwd
__device__ __forceinline__ int w512_sigma(int lane, int e) {
  const int k1 = lane >> 1, b = lane & 1, j = e & 7, c = e >> 3;
  return k1 + 16 * (8 * b + j + 16 * c);
}

}  // namespace idc
