// nd_internal.cuh -- pencil-kernel launchers shared by the 2D/3D drivers.
#pragma once
#include <cuda_runtime.h>

namespace idc {

// Blocked rank-major stream layout of the distributed 3D y passes (dist.cu):
// stream st (0..S-1) row l of local plane x at
//   base[input] + (l / L) * blk + st * soff + x * xstride + (l % L) * ncols.
// Passed to the launchers below, the backward pencils write their streams
// there (instead of in place / U) and the forward pencils read them from there.
struct DistLayout {
  double2* base[2];
  long L, nblocks, xstride, blk, soff;
  int S;
};

// K5: fftpadBackward on the m-row pencils of (batch x m x ncols) arrays f
// (and g if non-null): even stream in place, odd stream into U (V).
// odd_phase multiplies the odd stream (i^{-1} for the centered 4m transform
// fft0tpadBackward).
cudaError_t launch_pad_bwd(double2* f, double2* g, double2* U, double2* V, int m, long ncols, long batch,
                           long bstride, long ustride, cudaStream_t s, double2 odd_phase = double2{1.0, 0.0},
                           const DistLayout* dl = nullptr);
// K6: fftpadForward: f <- (FFT f + odd_phase zeta^{-k} FFT U)/(2m) (odd_phase = i
// for the centered 4m transform fft0tpadForward).
cudaError_t launch_pad_fwd(double2* f, const double2* U, int m, long ncols, long batch, long bstride, long ustride,
                           cudaStream_t s, double2 odd_phase = double2{1.0, 0.0}, const DistLayout* dl = nullptr);
// K7: centered fft0padBackward on (2m-1)-row pencils; streams in f (2m-1 rows) + U (m+1 rows).
cudaError_t launch_pad0_bwd(double2* f, double2* g, double2* U, double2* V, int m, long ncols, long batch,
                            long bstride, long ustride, cudaStream_t s, const DistLayout* dl = nullptr);
// K8: centered fft0padForward.
cudaError_t launch_pad0_fwd(double2* f, const double2* U, int m, long ncols, long batch, long bstride, long ustride,
                            cudaStream_t s, const DistLayout* dl = nullptr);

// TMA-staged persistent variants (pencils2.cu), 64 <= m <= 4096.
template <int N>
cudaError_t pad_bwd_tma(double2* f, double2* g, double2* U, double2* V, long ncols, long batch, long bstride,
                        long ustride, cudaStream_t s, double2 ophase, const DistLayout* dl = nullptr);
template <int N>
cudaError_t pad_fwd_tma(double2* f, const double2* U, long ncols, long batch, long bstride, long ustride,
                        cudaStream_t s, double2 ophase, const DistLayout* dl = nullptr);
template <int N>
cudaError_t pad0_bwd_tma(double2* f, double2* g, double2* U, double2* V, long ncols, long batch, long bstride,
                         long ustride, cudaStream_t s, const DistLayout* dl = nullptr);
template <int N>
cudaError_t pad0_fwd_tma(double2* f, const double2* U, long ncols, long batch, long bstride, long ustride,
                         cudaStream_t s, const DistLayout* dl = nullptr);

}  // namespace idc
