// launch.cu -- kernel launch + opt-in per-kernel-class profiler, see launch.cuh.
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/idconv.h"
#include "fft_dev.cuh"
#include "pdl.cuh"
#include "kernels.cuh"
#include "launch.cuh"

namespace idc {

namespace {
struct Rec {
  const char* tag;
  int n;
  long units;
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_free;   // recycled events

// transform counter: the per-translation-unit pointer setters (fft_dev.cuh)
std::vector<FftCounterSetter>& counter_setters() {
  static std::vector<FftCounterSetter> v;
  return v;
}
unsigned long long* g_counter = nullptr;

cudaEvent_t get_event() {
  if (!g_free.empty()) {
    cudaEvent_t e = g_free.back();
    g_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void register_fft_counter_setter(FftCounterSetter f) { counter_setters().push_back(f); }

cudaError_t launch_kernel(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t s,
                          const LaunchTag& tag) {
  count_launch();
  bool on;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    on = g_on;
  }
  // programmatic stream serialization: the kernel may be scheduled while the
  // previous kernel on the stream drains; its pdl_entry() waits (pdl.cuh)
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = IDC_PDL ? 1 : 0;
  if (!on) return cudaLaunchKernelExC(&cfg, fn, args);
  cudaEvent_t a, b;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    a = get_event();
    b = get_event();
  }
  cudaEventRecord(a, s);
  const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  cudaEventRecord(b, s);
  std::lock_guard<std::mutex> lk(g_mu);
  g_recs.push_back(Rec{tag.tag, tag.n, tag.units, a, b});
  return e;
}

Span span_begin(cudaStream_t s) {
  Span sp;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return sp;
  sp.a = get_event();
  cudaEventRecord(sp.a, s);
  return sp;
}

void span_end(Span& sp, cudaStream_t s, const LaunchTag& tag) {
  if (!sp.a) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t b = get_event();
  cudaEventRecord(b, s);
  g_recs.push_back(Rec{tag.tag, tag.n, tag.units, sp.a, b});
  sp.a = nullptr;
}

}  // namespace idc

extern "C" {

// Transform counter (instrumentation, debug library only): see fft_dev.cuh.
// begin zeroes the 16 counters (index log2 N) and arms every translation
// unit; end waits for the device, copies them to out[0..15] and disarms.
idc_status idc_fft_count_begin(void) {
  std::lock_guard<std::mutex> lk(idc::g_mu);
  if (idc::counter_setters().empty()) return IDC_ERR_UNSUPPORTED;   // product build: no counter code
  if (!idc::g_counter && cudaMalloc(&idc::g_counter, 16 * sizeof(unsigned long long)) != cudaSuccess) {
    idc::g_counter = nullptr;
    return IDC_ERR_CUDA;
  }
  if (cudaMemset(idc::g_counter, 0, 16 * sizeof(unsigned long long)) != cudaSuccess) return IDC_ERR_CUDA;
  for (auto f : idc::counter_setters())
    if (f(idc::g_counter) != cudaSuccess) return IDC_ERR_CUDA;
  return cudaDeviceSynchronize() == cudaSuccess ? IDC_OK : IDC_ERR_CUDA;
}

idc_status idc_fft_count_end(unsigned long long* out) {
  if (!out) return IDC_ERR_INVALID;
  std::lock_guard<std::mutex> lk(idc::g_mu);
  if (!idc::g_counter) return IDC_ERR_INVALID;
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(out, idc::g_counter, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return IDC_ERR_CUDA;
  for (auto f : idc::counter_setters())
    if (f(nullptr) != cudaSuccess) return IDC_ERR_CUDA;
  return cudaDeviceSynchronize() == cudaSuccess ? IDC_OK : IDC_ERR_CUDA;
}

idc_status idc_profile_begin(void) {
  std::lock_guard<std::mutex> lk(idc::g_mu);
  for (auto& r : idc::g_recs) {
    idc::g_free.push_back(r.a);
    idc::g_free.push_back(r.b);
  }
  idc::g_recs.clear();
  idc::g_on = true;
  return IDC_OK;
}

// Aggregates the records of the last begin..end window (once) and copies the
// text into buf; a second call with a larger buffer returns the same text.
long idc_profile_end(char* buf, size_t len) {
  static std::string last;
  static bool last_ok = true;
  std::vector<idc::Rec> recs;
  bool had;
  {
    std::lock_guard<std::mutex> lk(idc::g_mu);
    had = idc::g_on || !idc::g_recs.empty();
    idc::g_on = false;
    recs.swap(idc::g_recs);
  }
  if (had) {
    // (tag, n) -> launches, units, ms
    std::map<std::pair<std::string, int>, std::tuple<long, long, double>> agg;
    bool ok = true;
    for (auto& r : recs) {
      float ms = 0.f;
      if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) ok = false;
      auto& t = agg[{r.tag, r.n}];
      std::get<0>(t) += 1;
      std::get<1>(t) += r.units;
      std::get<2>(t) += ms;
    }
    {
      std::lock_guard<std::mutex> lk(idc::g_mu);
      for (auto& r : recs) {
        idc::g_free.push_back(r.a);
        idc::g_free.push_back(r.b);
      }
    }
    last.clear();
    char line[256];
    for (auto& kv : agg) {
      snprintf(line, sizeof line, "%s %d %ld %ld %.6f\n", kv.first.first.c_str(), kv.first.second,
               std::get<0>(kv.second), std::get<1>(kv.second), std::get<2>(kv.second));
      last += line;
    }
    last_ok = ok;
  }
  if (!last_ok) return -1;
  if (buf && len > 0) {
    const size_t n = last.size() < len - 1 ? last.size() : len - 1;
    last.copy(buf, n);
    buf[n] = 0;
  }
  return (long)last.size() + 1;
}

}  // extern "C"
