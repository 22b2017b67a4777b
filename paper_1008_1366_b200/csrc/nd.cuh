// nd.cuh -- 2D / 3D compositions (Functions cconv2, conv2, cconv3 and the
// Hermitian 3D analogue) built from the pencil kernels and the row kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace idc {

size_t cconv2d_work_bytes(size_t mx, size_t my, size_t batch);
size_t hconv2d_work_bytes(size_t mx, size_t my);
size_t cconv3d_work_bytes(size_t mx, size_t my, size_t mz);
size_t hconv3d_work_bytes(size_t mx, size_t my, size_t mz);

cudaError_t run_cconv2d(double2* f, double2* g, int mx, int my, long batch, double2* work, cudaStream_t s);
cudaError_t run_hconv2d(double2* f, double2* g, int mx, int my, double2* work, cudaStream_t s);
cudaError_t run_cconv3d(double2* f, double2* g, int mx, int my, int mz, double2* work, cudaStream_t s);
size_t hconv2d_dot_work_bytes(size_t npairs, size_t mx, size_t my);
size_t tconv2d_work_bytes(size_t mx, size_t my);
cudaError_t run_tconv2d(double2* f, double2* g, double2* h, int mx, int my, double2* work, cudaStream_t s);
size_t cconv2d_dot_work_bytes(size_t npairs, size_t mx, size_t my);
cudaError_t run_cconv2d_dot(double2* f, double2* g, int npairs, int mx, int my, double2* work, cudaStream_t s);
cudaError_t run_hconv2d_dot(double2* f, double2* g, int npairs, int mx, int my, double2* work, cudaStream_t s);
cudaError_t run_hconv3d(double2* f, double2* g, int mx, int my, int mz, double2* work, cudaStream_t s);

}  // namespace idc
