// tables.cuh -- plan-time roots of unity.
//
// zeta_N^k = exp(2 pi i k / N) for k < N, computed once per
// (device, N) on the host in long double with the integer argument reduced
// exactly, rounded to double and uploaded.  The paper factors zeta_N^k into
// two O(sqrt m) tables to save host cache; on the GPU a full
// table of N entries (<= 256 KiB) lives in L2/L1 and costs one 16-byte load
// per twiddle instead of a load plus a complex multiply (AMB-13: the two are
// equal to ~1 ulp).  Not timed: built on first use, outside every timed loop.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace idc {

// Device pointer to exp(+2 pi i k/N), k = 0..N-1, on the current device.
// Returns nullptr on failure (allocation / copy error).
const double2* zeta_table(int N);

// Device pointer to the Stockham pass-twiddle table of an N-point FFT with E
// elements per thread (layout: fft_dev.cuh, pass_tab_offset).  Same roots as
// zeta_table(N), regrouped so that a warp's twiddle loads are contiguous.
const double2* pass_table(int N, int E);

}  // namespace idc
