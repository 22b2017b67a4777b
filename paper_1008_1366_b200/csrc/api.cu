// api.cu -- the C ABI of include/idconv.h: validation, workspace queries and
// the composition of the hot-path kernels.  Host code only.
#include <cstdint>
#include <cstring>

#include "../../include/idconv.h"
#include "kernels.cuh"
#include "nd.cuh"

using idc::num_sms;

namespace {

bool is_pow2(size_t m) { return m >= 1 && (m & (m - 1)) == 0; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct Range {
  uintptr_t lo, hi;
};
Range rng(const void* p, size_t bytes) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  return {a, a + bytes};
}
bool overlap(Range a, Range b) { return a.lo < b.hi && b.lo < a.hi; }

idc_status from_cuda(cudaError_t e) { return e == cudaSuccess ? IDC_OK : IDC_ERR_CUDA; }

// common checks for 1..3 arrays of `bytes` each plus the workspace
idc_status check_arrays(const void* const* arrs, int n, size_t bytes, const void* work, size_t work_bytes,
                        size_t need) {
  for (int i = 0; i < n; ++i)
    if (!arrs[i] || !aligned16(arrs[i])) return IDC_ERR_INVALID;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (overlap(rng(arrs[i], bytes), rng(arrs[j], bytes))) return IDC_ERR_INVALID;
  if (need > 0) {
    if (!work || !aligned16(work)) return work ? IDC_ERR_INVALID : IDC_ERR_WORKSPACE;
    if (work_bytes < need) return IDC_ERR_WORKSPACE;
    for (int i = 0; i < n; ++i)
      if (overlap(rng(arrs[i], bytes), rng(work, need))) return IDC_ERR_INVALID;
  }
  return IDC_OK;
}

bool size_ok(size_t m, size_t lo, size_t hi) { return is_pow2(m) && m >= lo && m <= hi; }

}  // namespace

extern "C" {

const char* idc_status_string(idc_status s) {
  switch (s) {
    case IDC_OK: return "IDC_OK";
    case IDC_ERR_INVALID: return "IDC_ERR_INVALID: null/misaligned pointer, zero size or aliasing";
    case IDC_ERR_UNSUPPORTED: return "IDC_ERR_UNSUPPORTED: size outside the supported set";
    case IDC_ERR_WORKSPACE: return "IDC_ERR_WORKSPACE: workspace too small";
    case IDC_ERR_CUDA: return "IDC_ERR_CUDA: CUDA launch or runtime error";
    case IDC_ERR_NCCL: return "IDC_ERR_NCCL: NCCL error";
  }
  return "unknown idc_status";
}

const char* idc_version(void) { return "idconv 0.1 sm_100a fp64"; }

long long idc_launch_count(void) { return idc::launch_count(); }

size_t idc_workspace_bytes(idc_kind k, size_t m0, size_t m1, size_t m2, size_t batch) {
  switch (k) {
    case IDC_CCONV1D: return size_ok(m0, 1, 8192) ? idc::cconv_rows_work_bytes((int)m0) : 0;
    case IDC_HCONV1D: return size_ok(m0, 1, 8192) ? idc::hconv_rows_work_bytes((int)m0) : 0;
    case IDC_TCONV1D: return size_ok(m0, 1, 8192) ? idc::tconv_rows_work_bytes((int)m0) : 0;
    case IDC_CCONV2D: return idc::cconv2d_work_bytes(m0, m1, batch);
    case IDC_HCONV2D: return idc::hconv2d_work_bytes(m0, m1);
    case IDC_CCONV3D: return idc::cconv3d_work_bytes(m0, m1, m2);
    case IDC_HCONV3D: return idc::hconv3d_work_bytes(m0, m1, m2);
    case IDC_TCONV2D: return idc::tconv2d_work_bytes(m0, m1);
  }
  return 0;
}

idc_status idc_cconv1d(idc_c128* f, idc_c128* g, size_t m, size_t batch, void* work, size_t work_bytes,
                       idc_stream stream) {
  if (m == 0 || batch == 0) return IDC_ERR_INVALID;
  if (!size_ok(m, 1, 8192)) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  size_t need = idc::cconv_rows_work_bytes((int)m);
  idc_status st = check_arrays(arrs, 2, m * batch * sizeof(idc_c128), work, work_bytes, need);
  if (st != IDC_OK) return st;
  return from_cuda(idc::launch_cconv_rows(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)m,
                                          (long)batch, reinterpret_cast<double2*>(work), (cudaStream_t)stream));
}

idc_status idc_hconv1d(idc_c128* f, idc_c128* g, size_t m, size_t batch, void* work, size_t work_bytes,
                       idc_stream stream) {
  if (m == 0 || batch == 0) return IDC_ERR_INVALID;
  if (!size_ok(m, 1, 8192)) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  size_t need = idc::hconv_rows_work_bytes((int)m);
  idc_status st = check_arrays(arrs, 2, m * batch * sizeof(idc_c128), work, work_bytes, need);
  if (st != IDC_OK) return st;
  return from_cuda(idc::launch_hconv_rows(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)m,
                                          (long)batch, reinterpret_cast<double2*>(work), (cudaStream_t)stream));
}

idc_status idc_tconv1d(idc_c128* f, idc_c128* g, idc_c128* h, size_t m, size_t batch, void* work,
                       size_t work_bytes, idc_stream stream) {
  if (m == 0 || batch == 0) return IDC_ERR_INVALID;
  if (!size_ok(m, 1, 8192)) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g, h};
  size_t need = idc::tconv_rows_work_bytes((int)m);
  idc_status st = check_arrays(arrs, 3, m * batch * sizeof(idc_c128), work, work_bytes, need);
  if (st != IDC_OK) return st;
  return from_cuda(idc::launch_tconv_rows(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g),
                                          reinterpret_cast<double2*>(h), (int)m, (long)batch,
                                          reinterpret_cast<double2*>(work), (cudaStream_t)stream));
}

idc_status idc_cconv2d(idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t batch, void* work,
                       size_t work_bytes, idc_stream stream) {
  if (mx == 0 || my == 0 || batch == 0) return IDC_ERR_INVALID;
  if (!size_ok(mx, 1, 8192) || !size_ok(my, 1, 8192)) return IDC_ERR_UNSUPPORTED;
  size_t need = idc::cconv2d_work_bytes(mx, my, batch);
  if (need == 0) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  idc_status st = check_arrays(arrs, 2, mx * my * batch * sizeof(idc_c128), work, work_bytes, need);
  if (st != IDC_OK) return st;
  return from_cuda(idc::run_cconv2d(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)mx, (int)my,
                                    (long)batch, reinterpret_cast<double2*>(work), (cudaStream_t)stream));
}

idc_status idc_hconv2d(idc_c128* f, idc_c128* g, size_t mx, size_t my, void* work, size_t work_bytes,
                       idc_stream stream) {
  if (mx == 0 || my == 0) return IDC_ERR_INVALID;
  if (!size_ok(mx, 1, 8192) || !size_ok(my, 1, 8192)) return IDC_ERR_UNSUPPORTED;
  size_t need = idc::hconv2d_work_bytes(mx, my);
  if (need == 0) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  idc_status st = check_arrays(arrs, 2, (2 * mx - 1) * my * sizeof(idc_c128), work, work_bytes, need);
  if (st != IDC_OK) return st;
  return from_cuda(idc::run_hconv2d(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)mx, (int)my,
                                    reinterpret_cast<double2*>(work), (cudaStream_t)stream));
}

idc_status idc_tconv2d(idc_c128* f, idc_c128* g, idc_c128* h, size_t mx, size_t my, void* work,
                       size_t work_bytes, idc_stream stream) {
  if (mx == 0 || my == 0) return IDC_ERR_INVALID;
  if (!size_ok(mx, 1, 2048) || !size_ok(my, 1, 4096)) return IDC_ERR_UNSUPPORTED;
  size_t need = idc::tconv2d_work_bytes(mx, my);
  if (need == 0) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g, h};
  idc_status st = check_arrays(arrs, 3, 2 * mx * my * sizeof(idc_c128), work, work_bytes, need);
  if (st != IDC_OK) return st;
  return from_cuda(idc::run_tconv2d(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g),
                                    reinterpret_cast<double2*>(h), (int)mx, (int)my, reinterpret_cast<double2*>(work),
                                    (cudaStream_t)stream));
}

idc_status idc_cconv3d(idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t mz, void* work, size_t work_bytes,
                       idc_stream stream) {
  if (mx == 0 || my == 0 || mz == 0) return IDC_ERR_INVALID;
  if (!size_ok(mx, 1, 8192) || !size_ok(my, 1, 8192) || !size_ok(mz, 1, 8192)) return IDC_ERR_UNSUPPORTED;
  size_t need = idc::cconv3d_work_bytes(mx, my, mz);
  if (need == 0) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  idc_status st = check_arrays(arrs, 2, mx * my * mz * sizeof(idc_c128), work, work_bytes, need);
  if (st != IDC_OK) return st;
  return from_cuda(idc::run_cconv3d(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)mx, (int)my,
                                    (int)mz, reinterpret_cast<double2*>(work), (cudaStream_t)stream));
}

idc_status idc_hconv3d(idc_c128* f, idc_c128* g, size_t mx, size_t my, size_t mz, void* work, size_t work_bytes,
                       idc_stream stream) {
  if (mx == 0 || my == 0 || mz == 0) return IDC_ERR_INVALID;
  if (!size_ok(mx, 1, 8192) || !size_ok(my, 1, 8192) || !size_ok(mz, 1, 8192)) return IDC_ERR_UNSUPPORTED;
  size_t need = idc::hconv3d_work_bytes(mx, my, mz);
  if (need == 0) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  idc_status st =
      check_arrays(arrs, 2, (2 * mx - 1) * (2 * my - 1) * mz * sizeof(idc_c128), work, work_bytes, need);
  if (st != IDC_OK) return st;
  return from_cuda(idc::run_hconv3d(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)mx, (int)my,
                                    (int)mz, reinterpret_cast<double2*>(work), (cudaStream_t)stream));
}

// ---- multivector dot-product convolutions (NEXT-1) ----------

size_t idc_dot_workspace_bytes(idc_kind k, size_t npairs, size_t m0, size_t m1) {
  if (npairs == 0) return 0;
  if (k == IDC_HCONV2D) return idc::hconv2d_dot_work_bytes(npairs, m0, m1);
  if (k == IDC_CCONV2D) return idc::cconv2d_dot_work_bytes(npairs, m0, m1);
  return 0;   // 1D kinds need none
}

idc_status idc_cconv1d_dot(idc_c128* f, idc_c128* g, size_t npairs, size_t m, size_t batch, idc_stream stream) {
  if (m == 0 || batch == 0 || npairs == 0) return IDC_ERR_INVALID;
  if (!size_ok(m, 1, 4096)) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  idc_status st = check_arrays(arrs, 2, npairs * m * batch * sizeof(idc_c128), nullptr, 0, 0);
  if (st != IDC_OK) return st;
  return from_cuda(idc::launch_cconv_dot_rows(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g),
                                              (int)npairs, (long)(m * batch), (int)m, (long)batch,
                                              (cudaStream_t)stream));
}

idc_status idc_tconv1d_dot(idc_c128* f, idc_c128* g, idc_c128* h, size_t npairs, size_t m, size_t batch,
                           idc_stream stream) {
  if (m == 0 || batch == 0 || npairs == 0) return IDC_ERR_INVALID;
  if (!size_ok(m, 2, 4096)) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g, h};
  idc_status st = check_arrays(arrs, 3, npairs * m * batch * sizeof(idc_c128), nullptr, 0, 0);
  if (st != IDC_OK) return st;
  return from_cuda(idc::launch_tconv_dot_rows(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g),
                                              reinterpret_cast<double2*>(h), (int)npairs, (long)(m * batch), (int)m,
                                              (long)batch, (cudaStream_t)stream));
}

idc_status idc_cconv2d_dot(idc_c128* f, idc_c128* g, size_t npairs, size_t mx, size_t my, void* work,
                           size_t work_bytes, idc_stream stream) {
  if (mx == 0 || my == 0 || npairs == 0) return IDC_ERR_INVALID;
  if (!size_ok(mx, 1, 8192) || !size_ok(my, 1, 4096)) return IDC_ERR_UNSUPPORTED;
  size_t need = idc::cconv2d_dot_work_bytes(npairs, mx, my);
  if (need == 0) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  idc_status st = check_arrays(arrs, 2, npairs * mx * my * sizeof(idc_c128), work, work_bytes, need);
  if (st != IDC_OK) return st;
  return from_cuda(idc::run_cconv2d_dot(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)npairs,
                                        (int)mx, (int)my, reinterpret_cast<double2*>(work), (cudaStream_t)stream));
}

idc_status idc_hconv1d_dot(idc_c128* f, idc_c128* g, size_t npairs, size_t m, size_t batch, idc_stream stream) {
  if (m == 0 || batch == 0 || npairs == 0) return IDC_ERR_INVALID;
  if (!size_ok(m, 2, 4096)) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  idc_status st = check_arrays(arrs, 2, npairs * m * batch * sizeof(idc_c128), nullptr, 0, 0);
  if (st != IDC_OK) return st;
  return from_cuda(idc::launch_hconv_dot_rows(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g),
                                              (int)npairs, (long)(m * batch), (int)m, (long)batch,
                                              (cudaStream_t)stream));
}

idc_status idc_hconv2d_dot(idc_c128* f, idc_c128* g, size_t npairs, size_t mx, size_t my, void* work,
                           size_t work_bytes, idc_stream stream) {
  if (mx == 0 || my == 0 || npairs == 0) return IDC_ERR_INVALID;
  if (!size_ok(mx, 1, 8192) || !size_ok(my, 2, 4096)) return IDC_ERR_UNSUPPORTED;
  size_t need = idc::hconv2d_dot_work_bytes(npairs, mx, my);
  if (need == 0) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  idc_status st = check_arrays(arrs, 2, npairs * (2 * mx - 1) * my * sizeof(idc_c128), work, work_bytes, need);
  if (st != IDC_OK) return st;
  return from_cuda(idc::run_hconv2d_dot(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)npairs,
                                        (int)mx, (int)my, reinterpret_cast<double2*>(work), (cudaStream_t)stream));
}

idc_status idc_enforce_symmetry_2d(idc_c128* a, size_t mx, size_t my, size_t batch, idc_stream stream) {
  if (!a || !aligned16(a) || mx == 0 || my == 0 || batch == 0) return IDC_ERR_INVALID;
  return from_cuda(idc::launch_enforce_symmetry_2d(reinterpret_cast<double2*>(a), (int)mx, (int)my, (long)batch,
                                                   (cudaStream_t)stream));
}

size_t idc_advection2d_workspace_bytes(size_t mx, size_t my) {
  const size_t conv = idc::hconv2d_dot_work_bytes(2, mx, my);
  if (conv == 0) return 0;
  return conv + 3 * 2 * (2 * mx - 1) * my * sizeof(idc_c128);   // f (2 arrays), g (2 arrays), alignment slack
}

idc_status idc_advection2d(const idc_c128* w, idc_c128* out, size_t mx, size_t my, void* work, size_t work_bytes,
                           idc_stream stream) {
  if (!w || !out || mx == 0 || my == 0) return IDC_ERR_INVALID;
  if (!aligned16(w) || !aligned16(out) || (work && !aligned16(work))) return IDC_ERR_INVALID;
  if (!size_ok(mx, 1, 8192) || !size_ok(my, 2, 4096)) return IDC_ERR_UNSUPPORTED;
  const size_t need = idc_advection2d_workspace_bytes(mx, my);
  if (!work) return IDC_ERR_WORKSPACE;
  if (work_bytes < need) return IDC_ERR_WORKSPACE;
  const size_t n = (2 * mx - 1) * my;
  double2* F = reinterpret_cast<double2*>(work);
  double2* G = F + 2 * n;
  double2* cw = G + 2 * n;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = idc::launch_advection2d_inputs(reinterpret_cast<const double2*>(w), F, G, (int)mx, (int)my, s);
  if (e != cudaSuccess) return IDC_ERR_CUDA;
  e = idc::run_hconv2d_dot(F, G, 2, (int)mx, (int)my, cw, s);
  if (e != cudaSuccess) return IDC_ERR_CUDA;
  return from_cuda(cudaMemcpyAsync(out, F, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
}

// ---- general p/q implicit padding (NEXT-3) --------------------

idc_status idc_cconv1d_pq(idc_c128* f, idc_c128* g, size_t p, size_t q, size_t m, size_t batch, idc_stream stream) {
  if (m == 0 || batch == 0 || p == 0 || q == 0) return IDC_ERR_INVALID;
  if (p > 3 || q > 8 || q < 2 * p || !size_ok(m, 8, 2048)) return IDC_ERR_UNSUPPORTED;
  const void* arrs[] = {f, g};
  idc_status st = check_arrays(arrs, 2, p * m * batch * sizeof(idc_c128), nullptr, 0, 0);
  if (st != IDC_OK) return st;
  return from_cuda(idc::launch_cconv_pq_rows(reinterpret_cast<double2*>(f), reinterpret_cast<double2*>(g), (int)p,
                                             (int)q, (int)m, (long)batch, (cudaStream_t)stream));
}

}  // extern "C"
