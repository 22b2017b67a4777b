// dist.cu -- distributed 3D driver over NCCL (placeholder until K10 lands).
#include "../../include/idconv.h"

extern "C" {
idc_status idc_comm_init(void** comm, int, int, const void*) {
  if (comm) *comm = nullptr;
  return IDC_ERR_UNSUPPORTED;
}
idc_status idc_comm_destroy(void*) { return IDC_OK; }
idc_status idc_comm_unique_id(void*) { return IDC_ERR_UNSUPPORTED; }
size_t idc_dist_workspace_bytes(idc_kind, size_t, size_t, size_t, int) { return 0; }
idc_status idc_cconv3d_dist(void*, idc_c128*, idc_c128*, size_t, size_t, size_t, void*, size_t, idc_stream) {
  return IDC_ERR_UNSUPPORTED;
}
}
