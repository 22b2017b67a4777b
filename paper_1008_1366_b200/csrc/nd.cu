// nd.cu -- 2D / 3D compositions (placeholder until the pencil kernels land).
#include "nd.cuh"

namespace idc {
size_t cconv2d_work_bytes(size_t, size_t, size_t) { return 0; }
size_t hconv2d_work_bytes(size_t, size_t) { return 0; }
size_t cconv3d_work_bytes(size_t, size_t, size_t) { return 0; }
size_t hconv3d_work_bytes(size_t, size_t, size_t) { return 0; }
cudaError_t run_cconv2d(double2*, double2*, int, int, long, double2*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t run_hconv2d(double2*, double2*, int, int, double2*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t run_cconv3d(double2*, double2*, int, int, int, double2*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t run_hconv3d(double2*, double2*, int, int, int, double2*, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace idc
