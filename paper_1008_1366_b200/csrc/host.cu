// host.cu -- host-buffer execution of the batched 1D convolutions: the rows
// are streamed through the device in chunks on a small pool of streams so
// that the host->device copy of chunk c+1, the fused row kernel of chunk c
// and the device->host copy of chunk c-1 overlap (copy engines and SMs work
// concurrently).  Plumbing around the hot path (no arithmetic here); the
// kernels are the same K2/K3/K4 launches as idc_{c,h,t}conv1d.
#include <cstdint>
#include <mutex>

#include "../../include/idconv.h"
#include "kernels.cuh"

namespace {

constexpr int kSlots = 3;

struct HostPool {
  cudaStream_t s[kSlots];
  cudaEvent_t fork, done[kSlots];
  std::mutex enq;      // held from the fork record to the last join: concurrent
                       // host threads must not interleave their fork/join events
  bool ok = false;
};

HostPool& host_pool() {
  static HostPool p[16];
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  HostPool& q = p[dev & 15];
  if (!q.ok) {
    for (int i = 0; i < kSlots; ++i) {
      cudaStreamCreateWithFlags(&q.s[i], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&q.done[i], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&q.fork, cudaEventDisableTiming);
    q.ok = true;
  }
  return q;
}

int n_inputs(idc_kind k) { return k == IDC_TCONV1D ? 3 : 2; }

size_t row_work(idc_kind k, int m) {
  switch (k) {
    case IDC_CCONV1D: return idc::cconv_rows_work_bytes(m);
    case IDC_HCONV1D: return idc::hconv_rows_work_bytes(m);
    case IDC_TCONV1D: return idc::tconv_rows_work_bytes(m);
    default: return 0;
  }
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Rows of the next chunk.  The pipeline's first host->device copy and last
// device->host copy overlap nothing, so chunks ramp up from chunk/8 rows
// (doubling) and the last 2*chunk rows are cut into halving pieces (down to
// chunk/8): the exposed fill and drain shrink to about 1/8 of a chunk each.
size_t next_chunk(size_t done, size_t batch, size_t chunk, size_t index) {
  const size_t rem = batch - done;
  const size_t small = chunk / 8 > 0 ? chunk / 8 : 1;
  size_t c = chunk;
  if (index < 3) c = small << index;                      // chunk/8, chunk/4, chunk/2, then chunk
  if (c > chunk) c = chunk;
  if (rem < 2 * chunk) {
    const size_t half = (rem + 1) / 2;
    if (half < c) c = half;
  }
  if (c < small) c = small;
  if (c > rem) c = rem;
  return c;
}

}  // namespace

extern "C" {

size_t idc_host_workspace_bytes(idc_kind k, size_t m, size_t chunk_rows) {
  if (k != IDC_CCONV1D && k != IDC_HCONV1D && k != IDC_TCONV1D) return 0;
  if (m < 1 || m > 8192 || (m & (m - 1)) != 0 || chunk_rows == 0) return 0;
  const size_t arr = align256(chunk_rows * m * sizeof(idc_c128));
  return kSlots * (n_inputs(k) * arr + align256(row_work(k, (int)m)));
}

idc_status idc_conv1d_host(idc_kind k, const idc_c128* const* in_host, idc_c128* out_host, size_t m, size_t batch,
                           size_t chunk_rows, void* work, size_t work_bytes, idc_stream stream) {
  if (!in_host || !out_host || m == 0 || batch == 0 || chunk_rows == 0) return IDC_ERR_INVALID;
  if (k != IDC_CCONV1D && k != IDC_HCONV1D && k != IDC_TCONV1D) return IDC_ERR_UNSUPPORTED;
  const int nin = n_inputs(k);
  for (int i = 0; i < nin; ++i)
    if (!in_host[i]) return IDC_ERR_INVALID;
  const size_t need = idc_host_workspace_bytes(k, m, chunk_rows);
  if (need == 0) return IDC_ERR_UNSUPPORTED;
  if (!work) return IDC_ERR_WORKSPACE;
  if (work_bytes < need) return IDC_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(work) & 255u) != 0) return IDC_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  HostPool& P = host_pool();
  std::lock_guard<std::mutex> enq(P.enq);
  const size_t arr = align256(chunk_rows * m * sizeof(idc_c128));
  const size_t per_slot = nin * arr + align256(row_work(k, (int)m));
  if (cudaEventRecord(P.fork, s) != cudaSuccess) return IDC_ERR_CUDA;
  for (int i = 0; i < kSlots; ++i)
    if (cudaStreamWaitEvent(P.s[i], P.fork, 0) != cudaSuccess) return IDC_ERR_CUDA;
  size_t c = 0;
  for (size_t r0 = 0, rows = 0; r0 < batch; r0 += rows, ++c) {
    rows = next_chunk(r0, batch, chunk_rows, c);
    const int slot = (int)(c % kSlots);
    cudaStream_t st = P.s[slot];
    char* base = static_cast<char*>(work) + slot * per_slot;
    double2* d[3];
    for (int i = 0; i < nin; ++i) {
      d[i] = reinterpret_cast<double2*>(base + i * arr);
      if (cudaMemcpyAsync(d[i], in_host[i] + r0 * m, rows * m * sizeof(idc_c128), cudaMemcpyHostToDevice, st) !=
          cudaSuccess)
        return IDC_ERR_CUDA;
    }
    double2* rw = reinterpret_cast<double2*>(base + nin * arr);
    cudaError_t e;
    if (k == IDC_CCONV1D) e = idc::launch_cconv_rows(d[0], d[1], (int)m, (long)rows, rw, st);
    else if (k == IDC_HCONV1D) e = idc::launch_hconv_rows(d[0], d[1], (int)m, (long)rows, rw, st);
    else e = idc::launch_tconv_rows(d[0], d[1], d[2], (int)m, (long)rows, rw, st);
    if (e != cudaSuccess) return IDC_ERR_CUDA;
    if (cudaMemcpyAsync(out_host + r0 * m, d[0], rows * m * sizeof(idc_c128), cudaMemcpyDeviceToHost, st) !=
        cudaSuccess)
      return IDC_ERR_CUDA;
  }
  for (int i = 0; i < kSlots; ++i) {
    if (cudaEventRecord(P.done[i], P.s[i]) != cudaSuccess) return IDC_ERR_CUDA;
    if (cudaStreamWaitEvent(s, P.done[i], 0) != cudaSuccess) return IDC_ERR_CUDA;
  }
  return IDC_OK;
}

}  // extern "C"
