// kernels.cuh -- launchers of the fused hot-path kernels (host side).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace idc {

// Bytes of global stash the row kernels need for rows of length m (0 when the
// stash fits in shared memory).
size_t cconv_rows_work_bytes(int m);
size_t hconv_rows_work_bytes(int m);
size_t tconv_rows_work_bytes(int m);

// K2: Function cconv on `nrows` independent row pairs
// (f + r*ldf, g + r*ldg), rows of m complex, result in f.
cudaError_t launch_cconv_rows(double2* f, double2* g, int m, long nrows, double2* work, cudaStream_t s);

// K3: centered Hermitian conv (P:529-554 / Function conv) on rows.
cudaError_t launch_hconv_rows(double2* f, double2* g, int m, long nrows, double2* work, cudaStream_t s);

// K4: centered Hermitian ternary conv (Function tconv) on rows.
cudaError_t launch_tconv_rows(double2* f, double2* g, double2* h, int m, long nrows, double2* work,
                              cudaStream_t s);

// Two row sets in one launch: rows [0, n0) are rows of (f, g), rows
// [n0, nrows) are rows of (f1, g1) -- the two residue streams of an outer
// implicit transform (Functions cconv2 / conv2 run cconv / conv on both),
// one launch instead of two (better wave balance, one fewer launch).
struct RowSets {
  double2* f1 = nullptr;
  double2* g1 = nullptr;
  long n0 = -1;       // < 0: one set
};
__host__ __device__ inline double2* row_ptr(double2* a0, double2* a1, long n0, long row, int m) {
  return (n0 < 0 || row < n0) ? a0 + row * (long)m : a1 + (row - n0) * (long)m;
}
cudaError_t launch_cconv_rows_sets(double2* f, double2* g, long n0, double2* f1, double2* g1, long n1, int m,
                                   double2* work, cudaStream_t s);
cudaError_t launch_hconv_rows_sets(double2* f, double2* g, long n0, double2* f1, double2* g1, long n1, int m,
                                   double2* work, cudaStream_t s);

// Register-resident variants (rows2.cu), m <= 4096.
template <int M> cudaError_t cconv_rows2(double2* f, double2* g, long nrows, cudaStream_t s, RowSets rs = {});
template <int M> cudaError_t hconv_rows2(double2* f, double2* g, long nrows, cudaStream_t s);
template <int M> cudaError_t tconv_rows2(double2* f, double2* g, double2* h, long nrows, cudaStream_t s);

// TMA-staged Hermitian / ternary variants (rows3.cu), 512 <= m <= 4096.
template <int M> cudaError_t hconv_rows3(double2* f, double2* g, long nrows, cudaStream_t s, RowSets rs = {});
template <int M> cudaError_t tconv_rows3(double2* f, double2* g, double2* h, long nrows, cudaStream_t s);

// K3d (rows_dot.cu): centered Hermitian dot-product convolution of npairs
// row pairs (pair i at f + i*istride, g + i*istride), result in pair 0.
cudaError_t launch_hconv_dot_rows(double2* f, const double2* g, int npairs, long istride, int m, long nrows,
                                  cudaStream_t s);
// K2d / K4d (rows_dot.cu): complex and ternary dot products, same layout.
cudaError_t launch_cconv_dot_rows(double2* f, const double2* g, int npairs, long istride, int m, long nrows,
                                  cudaStream_t s);
cudaError_t launch_tconv_dot_rows(double2* f, const double2* g, const double2* h, int npairs, long istride, int m,
                                  long nrows, cudaStream_t s);
// K2pq (rows_dot.cu): complex rows of p*m modes implicitly padded to q*m.
cudaError_t launch_cconv_pq_rows(double2* f, const double2* g, int p, int q, int m, long nrows, cudaStream_t s);
// Hermitian projection of the ky = 0 lines of batch (2mx-1) x my arrays.
cudaError_t launch_enforce_symmetry_2d(double2* a, int mx, int my, long batch, cudaStream_t s);
// The four M = 2 inputs of the 2D Euler advective term from w.
cudaError_t launch_advection2d_inputs(const double2* w, double2* f, double2* g, int mx, int my, cudaStream_t s);

// Count of hot-path kernel launches issued by this library (every launcher
// calls count_launch() right before cudaLaunchKernel); read through the ABI
// as idc_launch_count() so a benchmark can report its own kernel launches.
void count_launch();
long long launch_count();

// Number of SMs of the current device (cached).
int num_sms();

}  // namespace idc
