// tmap.cu -- cuTensorMapEncodeTiled through the runtime's driver entry point
// (no link-time dependency on libcuda).
#include <cudaTypedefs.h>

#include <mutex>

#include "tmap.cuh"

namespace idc {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_once;
void load_entry() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}
}  // namespace

bool encode_pencil_map(CUtensorMap* map, const void* base, long ncols, long rows, long batch, long bstride, int W,
                       int BR, bool swizzle128) {
  if (swizzle128 && W * 16 != 128) return false;
  std::call_once(g_once, load_entry);
  if (!g_encode) return false;
  // fp64 elements; the innermost dimension interleaves (re, im)
  cuuint64_t dims[3] = {(cuuint64_t)(2 * ncols), (cuuint64_t)rows, (cuuint64_t)(batch < 1 ? 1 : batch)};
  cuuint64_t strides[2] = {(cuuint64_t)(ncols * 16), (cuuint64_t)((batch > 1 ? bstride : rows * ncols) * 16)};
  cuuint32_t box[3] = {(cuuint32_t)(2 * W), (cuuint32_t)BR, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_blocked_map(CUtensorMap* map, const void* base, long ncols, long L, long nx, long nblocks, long xstride,
                        long blk, int W, int BR) {
  std::call_once(g_once, load_entry);
  if (!g_encode || BR > L) return false;
  cuuint64_t dims[4] = {(cuuint64_t)(2 * ncols), (cuuint64_t)L, (cuuint64_t)nx, (cuuint64_t)nblocks};
  cuuint64_t strides[3] = {(cuuint64_t)(ncols * 16), (cuuint64_t)(xstride * 16), (cuuint64_t)(blk * 16)};
  cuuint32_t box[4] = {(cuuint32_t)(2 * W), (cuuint32_t)BR, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace idc
